"""B200-native GCA-H2 hot path for Laplace BEM (arXiv:1810.08429).

A drop-in for the hot path of the reference package ``greencross``: the
modules mirror its public API (geometry, quadrature, clustering, assembly,
gca, h2, cli.build_h2_operator) while batched FP64 quadrature, Green
factors, cross approximation and the H2 matvec run as sm_100a kernels in
``libgcb200.so`` (C-ABI: include/gcb200.h).
"""

__version__ = "0.1.0"

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native kernels")


def golden(name):
    with np.load(os.path.join(GOLDEN, name)) as f:
        return {k: f[k] for k in f.files}


@pytest.fixture(scope="session")
def sphere2():
    from paper_1810_08429_b200.geometry import build_sphere_mesh
    return build_sphere_mesh(2)


@pytest.fixture(scope="session")
def sphere3():
    from paper_1810_08429_b200.geometry import build_sphere_mesh
    return build_sphere_mesh(3)


def mesh_for(name):
    from paper_1810_08429_b200.geometry import build_cube_mesh, build_sphere_mesh
    tag = name.split("_")[1].split(".")[0]          # e.g. sphere4, cube3
    kind, level = tag[:-1], int(tag[-1])
    return build_sphere_mesh(level) if kind == "sphere" else build_cube_mesh(level)


PIPELINES = ["h2_sphere4_eps1e-4.npz", "h2_cube4_eps1e-6.npz", "h2_sphere5_eps1e-6.npz"]


def eps_of(name):
    return float(name.split("_eps")[1][:-4])

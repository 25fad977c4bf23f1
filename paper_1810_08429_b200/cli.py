"""Operator construction shared by the experiment driver (``cli.py:159-177``).

Only the configuration record, ``build_h2_operator`` - the canonical
assembly sequence the benchmark reproduces - and the executor statistics
report of ``greencross stats`` are mirrored; the rest of the CSV experiment
driver is out of scope.
"""

import csv
from collections import namedtuple

import numpy as np

from . import gca
from .clustering import build_block_tree, build_cluster_tree
from .errors import ConfigError

STATS_COLUMNS = ["case", "batches", "tasks", "wall_s"]          # cli.py:42-43
CASE_NAMES = ("disjoint", "vertex", "edge", "identical")

ExperimentConfig = namedtuple("ExperimentConfig", [
    "level", "geometry", "basis", "disc", "eta", "m", "delta_factor",
    "eps", "leaf_size", "q_reg", "q_sing", "lam", "source", "seed"])


def default_config(**kw):
    """CLI defaults (``cli.py:411-449``): eta 1, m 3, delta 0.5, eps 1e-4,
    leaf 16, q = (3, 5)."""
    base = dict(level=4, geometry="plane", basis="constant", disc="galerkin", eta=1.0,
                m=3, delta_factor=0.5, eps=1e-4, leaf_size=16, q_reg=3, q_sing=5,
                lam=0.5, source=(2.0, 0.0, 0.0), seed=0)
    base.update(kw)
    return validate_config(ExperimentConfig(**base))


def validate_config(cfg):
    if not 0.0 < cfg.lam < 1.0:
        raise ConfigError("lambda must lie in (0, 1), got %g" % cfg.lam)
    if np.linalg.norm(cfg.source) <= 1.0:
        raise ConfigError("source point must lie strictly outside the closed unit ball")
    if cfg.eta <= 0.0:
        raise ConfigError("eta must be positive")
    if cfg.m < 1:
        raise ConfigError("green order m must be at least 1")
    if cfg.eps <= 0.0:
        raise ConfigError("aca eps must be positive")
    if cfg.delta_factor <= 0.0:
        raise ConfigError("delta factor must be positive")
    if cfg.leaf_size < 1:
        raise ConfigError("leaf size must be at least 1")
    if min(cfg.q_reg, cfg.q_sing) < 1:
        raise ConfigError("quadrature orders must be at least 1")
    if cfg.disc == "collocation" and cfg.basis != "linear":
        raise ConfigError("collocation pairs with the linear basis only")
    return cfg


def build_h2_operator(mesh, cfg, kind="slp", capacity=None, threads=None, device=None,
                      timings=None):
    """Cluster tree, block tree and GCA-H2 matrix for one configuration;
    returns ``(h2matrix, tree, btree)`` like ``cli.py:159-177``.  When a dict
    is passed as ``timings`` it receives the host/device phase times."""
    import time

    from .device import require_device
    dev = require_device(device)
    t0 = time.perf_counter()
    tree = build_cluster_tree(mesh, basis_kind=cfg.basis, leaf_size=cfg.leaf_size, device=dev)
    t1 = time.perf_counter()
    btree = build_block_tree(tree, eta=cfg.eta)
    t2 = time.perf_counter()
    orders = (cfg.q_reg, cfg.q_sing)
    rmarks, cmarks = gca.coupling_mark_arrays(btree)
    # row and column bases in shared per-level launches (gca.build_cluster_bases)
    row_kind = "collocation" if cfg.disc == "collocation" else cfg.basis      # cli.py:167
    rb, cb = gca.build_cluster_bases(tree, mesh, cfg.basis, cfg.m, cfg.delta_factor, cfg.eps,
                                     [("row", rmarks, row_kind), ("col", cmarks, cfg.basis)], orders,
                                     device)
    t3 = t4 = time.perf_counter()
    hm = gca.build_h2(btree, rb, cb, mesh, kind=kind, basis=cfg.basis, disc=cfg.disc,
                      orders=orders, device=device)
    t5 = time.perf_counter()
    if timings is not None:
        timings.update(cluster_tree_s=t1 - t0, block_tree_s=t2 - t1, row_basis_s=t3 - t2,
                       col_basis_s=t4 - t3, build_h2_s=t5 - t4, total_s=t5 - t0)
    return hm, tree, btree


def stats_rows(hm):
    """The rows of ``greencross stats`` (``cli.py:389-404``) for one built
    operator: case name, capacity-sealed batches, tasks, evaluator seconds."""
    return [{"case": CASE_NAMES[st["case"]], "batches": st["batches"], "tasks": st["tasks"],
             "wall_s": st["wall_s"]} for st in hm.exec_stats]


def write_stats(path, hm):
    """``stats_rows`` as the reference's CSV report (header STATS_COLUMNS)."""
    rows = stats_rows(hm)
    with open(path, "w", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=STATS_COLUMNS)
        writer.writeheader()
        for row in rows:
            writer.writerow(row)
    return rows

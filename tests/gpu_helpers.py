"""Shared set-up for the GPU parity tests: build a context from an ie_workloads config and
compute the matching oracle quantities.  (Test infrastructure; imports both sides.)"""

import numpy as np

from ie_workloads import make_config
from oracle import physics


def gpu_ctx(cfg, sigma=None, nrhs=None, boxes=None, restart=None):
    import torch
    import paper_2306_17537_b200 as ie
    sigma = cfg.sigma() if sigma is None else sigma
    ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
    ie.ensure_workspace(ctx, boxes=boxes if boxes is not None else cfg.boxes,
                        nrhs=nrhs or max(1, len(cfg.sources)), restart=restart or cfg.restart)
    ie.ie_set_contrast(ctx, torch.from_numpy(np.ascontiguousarray(sigma)).cuda())
    if cfg.sources:
        ie.ie_set_source(ctx, np.array([s for s, _ in cfg.sources]), np.array([m for _, m in cfg.sources]))
    return ctx, sigma


def oracle_setup(cfg, sigma):
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(sigma, cfg.sigma_b)
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    E0 = np.ascontiguousarray(np.stack([np.moveaxis(physics.incident_E(pts, s, m, k0, cfg.freq), -1, 0)
                                        for s, m in cfg.sources])) if cfg.sources else None
    return k0, ds, E0


def rel(a, b):
    """Relative L2 error; for an all-zero reference the absolute L2 norm of a (must be 0-ish)."""
    nb = np.linalg.norm(np.asarray(b).ravel())
    d = np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel())
    return float(d / nb) if nb > 0 else float(d)


__all__ = ["gpu_ctx", "oracle_setup", "rel", "make_config"]

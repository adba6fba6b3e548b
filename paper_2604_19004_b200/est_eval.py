"""Estimation-accuracy harness on the GPU.

Restates the reference's ``est-eval`` command (cli.py:301-341) without its
file I/O: for every register count it runs the FORCE_ESTIMATE workflow with
``compute_estimation_errors`` (engine.py:218-226, reduced on the device by
``sg_est_errors``) and records the same fields as the reference CSV rows,
plus the sampled-CR error the paper reports (§5.3).
"""

from __future__ import annotations

from dataclasses import replace

from .config import EngineConfig, WorkflowOverride


def est_eval(a, b=None, op: str = "aa", registers=(32, 64, 128), cfg: EngineConfig | None = None,
             name: str = "") -> list:
    """One record per register count (reference cmd_est_eval field names)."""
    from . import multiply_mode
    from .engine import spgemm
    if any(r not in (32, 64, 128) for r in registers):
        raise ValueError("register counts must be 32, 64 or 128")
    base = cfg or EngineConfig()
    a2, b2 = multiply_mode(a, op, b)
    out = []
    for m in registers:
        c = replace(base, workflow=WorkflowOverride.FORCE_ESTIMATE, registers=m, compute_estimation_errors=True,
                    return_device=True)
        res, rep = spgemm(a2, b2, c)
        del res
        nrows = a2.nrows
        cr_err = None
        if rep.cr_hat is not None and rep.cr_true:
            cr_err = abs(rep.cr_hat - rep.cr_true) / rep.cr_true
        out.append({
            "matrix": name, "op": op, "workflow": "estimate", "registers": m,
            "coef": "" if base.coef is None else base.coef, "seed": base.seed, "status": "ok",
            "nnz_a": a2.nnz, "nnz_c": rep.nnz_c, "products": rep.total_products,
            "flops": 2 * rep.total_products, "overflow_rows": rep.overflow_row_count,
            "overflow_ratio": rep.overflow_row_count / nrows if nrows else 0.0,
            "mean_rel_err": rep.est_mean_rel_err, "std_rel_err": rep.est_std_rel_err,
            "cr_true": "" if rep.cr_true is None else rep.cr_true,
            "cr_sampled": "" if rep.cr_hat is None else rep.cr_hat,
            "cr_sampled_rel_err": cr_err, "gpu_ms": rep.total_ms,
        })
    return out

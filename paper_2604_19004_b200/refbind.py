"""Reference-side binding: run the reference package's ``spgemm`` on the B200.

This is the switch INTEGRATION.md §2 describes, as code a maintainer of the
reference package (``sketchgemm``) would import.  ``bind(sketchgemm)``
returns a function with the reference signature
``spgemm(a, b, cfg=None, deadline=None) -> (CsrMatrix, RunReport)``
(reference ``engine.py:136-137``) that:

* forwards EVERY ``EngineConfig`` field (``engine.py:54-74``): workflow,
  registers, tiers (all ``TierConfig`` fields, ``accumulate.py:47-71``),
  coef, sample_ratio / sample_min / sample_max, seed, workers,
  staging_limit_bytes, compute_estimation_errors;
* returns the reference's own ``CsrMatrix`` and ``RunReport`` types, with
  the reference's report fields only;
* raises the reference's own ``ResourceLimitError`` / ``DeadlineExceeded``
  (``engine.py:39-44``) and ``ValueError`` for dimension mismatches.

``install(sketchgemm)`` rebinds ``sketchgemm.spgemm`` and
``sketchgemm.engine.spgemm`` to it, so the reference's own tests run against
the GPU path unchanged (tests/test_gpu_reference_suite.py).
"""

from __future__ import annotations

import dataclasses

from . import config as _cfg
from .engine import spgemm as _spgemm

_REPORT_FIELDS = None


def engine_config(ref_cfg) -> _cfg.EngineConfig:
    """The B200 EngineConfig for a reference EngineConfig (or None)."""
    if ref_cfg is None:
        return _cfg.EngineConfig(deterministic=True)
    t = ref_cfg.tiers
    tiers = _cfg.TierConfig(hash_capacities=tuple(t.hash_capacities),
                            enhanced_hash_capacity=int(t.enhanced_hash_capacity),
                            dense_spans=tuple(t.dense_spans),
                            esc_max_products=int(t.esc_max_products),
                            expansion_coef=float(t.expansion_coef),
                            bitmap_query_threshold=float(t.bitmap_query_threshold))
    return _cfg.EngineConfig(
        workflow=_cfg.WorkflowOverride(ref_cfg.workflow.value),
        registers=ref_cfg.registers,
        tiers=tiers,
        coef=ref_cfg.coef,
        sample_ratio=ref_cfg.sample_ratio,
        sample_min=ref_cfg.sample_min,
        sample_max=ref_cfg.sample_max,
        seed=ref_cfg.seed,
        workers=ref_cfg.workers,
        staging_limit_bytes=ref_cfg.staging_limit_bytes,
        compute_estimation_errors=ref_cfg.compute_estimation_errors,
        # the reference's contract includes bit-identical values for a fixed
        # seed at any worker count (engine.py:13-14)
        deterministic=True)


def bind(sg):
    """spgemm with the reference signature and types, computed on the GPU."""
    ref_fields = [f.name for f in dataclasses.fields(sg.RunReport)]

    def spgemm(a, b, cfg=None, deadline=None):
        ours = engine_config(cfg)
        try:
            c, rep = _spgemm(a, b, ours, deadline)
        except _cfg.ResourceLimitError as exc:
            raise sg.ResourceLimitError(str(exc)) from exc
        except _cfg.DeadlineExceeded as exc:
            raise sg.DeadlineExceeded(str(exc)) from exc
        C = sg.CsrMatrix(c.nrows, c.ncols, c.row_ptr, c.col_idx, c.values)
        R = sg.RunReport(**{k: getattr(rep, k) for k in ref_fields})
        return C, R

    spgemm.__doc__ = "B200 spgemm bound to the reference types (paper_2604_19004_b200.refbind)."
    return spgemm


def install(sg):
    """Route the reference package's spgemm to the GPU path."""
    fn = bind(sg)
    sg.spgemm = fn
    sg.engine.spgemm = fn
    return fn

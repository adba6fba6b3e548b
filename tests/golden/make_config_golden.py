"""Config-scale golden fixtures from the REAL reference (build container only).

    PYTHONPATH=. python tests/golden/make_config_golden.py [poisson64 rect rmat20]

Runs ``sketchgemm.spgemm`` (imported read-only from /root/reference/pkg/src)
on the BASELINE configs at their real size:

  * poisson64 (configs[1]) and rect (configs[3]) whole;
  * rmat20 (configs[2]) on the 20 products-stratified row blocks of
    ``matgen.stratified_blocks`` (2.05% of its 2.09e10 products, hub rows
    first) -- the whole product needs ~0.9 TB of host memory in the
    reference, and rows are independent (engine.py:13-14).

C is too large to commit, so each fixture keeps what pins it:
  * sha256 of row_ptr and col_idx (structure is bit-exact by contract);
  * value sums over consecutive groups of GROUP entries (all values are
    positive, so each group sum is within the per-entry rtol 1e-12);
  * every entry of a few sampled rows (per-entry rtol 1e-12);
  * the RunReport fields (whole-matrix configs).
tests/test_gpu_config_scale.py compares the GPU C with these, and with the
oracle port on the same rows at run time.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, f"{REF}/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import sketchgemm as sg  # noqa: E402

from paper_2604_19004_b200 import matgen  # noqa: E402

OUT = os.path.join(HERE, "configs")
GROUP = 4096


def sha(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def group_sums(v: np.ndarray, g: int = GROUP) -> np.ndarray:
    n = len(v)
    if n == 0:
        return np.zeros(0)
    return np.add.reduceat(v, np.arange(0, n, g))


def ref_csr(a):
    return sg.CsrMatrix(a.nrows, a.ncols, np.asarray(a.row_ptr), np.asarray(a.col_idx), np.asarray(a.values))


def pin(c, rng, nsample=64):
    """Fixture fields of one C (or C block)."""
    rp, ci, vv = c.row_ptr, c.col_idx, c.values
    live = np.flatnonzero(np.diff(rp) > 0)
    pick = np.sort(rng.choice(live, size=min(nsample, len(live)), replace=False)) if len(live) else live
    # keep sampled rows bounded (hub rows hold ~0.5 M entries): at most 4096
    # entries of each sampled row, taken from its start
    cols, vals, lens = [], [], []
    for r in pick:
        s, e = int(rp[r]), int(rp[r + 1])
        e = min(e, s + 4096)
        cols.append(ci[s:e])
        vals.append(vv[s:e])
        lens.append(e - s)
    return {
        "meta": {"nrows": int(c.nrows), "ncols": int(c.ncols), "nnz": int(rp[-1]),
                 "sha_row_ptr": sha(rp.astype(np.int64)), "sha_col_idx": sha(ci.astype(np.int32)),
                 "group": GROUP},
        "arrays": {"group_sums": group_sums(vv), "sample_rows": pick.astype(np.int64),
                   "sample_lens": np.asarray(lens, np.int64),
                   "sample_cols": np.concatenate(cols) if cols else np.zeros(0, np.int32),
                   "sample_vals": np.concatenate(vals) if vals else np.zeros(0)},
    }


def save(name, meta, arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    with open(os.path.join(OUT, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def whole(name):
    a, b = matgen.make_config(name)
    t0 = time.perf_counter()
    c, rep = sg.spgemm(ref_csr(a), ref_csr(b), sg.EngineConfig(workers=os.cpu_count() or 1, seed=0))
    dt = time.perf_counter() - t0
    p = pin(c, np.random.default_rng(1))
    p["meta"]["report"] = {k: v for k, v in dataclasses.asdict(rep).items() if not k.endswith("_ms")}
    p["meta"]["reference_seconds"] = dt
    p["meta"]["workers"] = os.cpu_count()
    save(name, p["meta"], p["arrays"])
    print(f"{name}: nnz {rep.nnz_c} workflow {rep.workflow} in {dt:.1f}s", flush=True)


def rmat20_blocks():
    a, b = matgen.make_config("rmat20")
    per = matgen.row_products(a, b)
    blocks = matgen.stratified_blocks(per)
    bref = ref_csr(b)
    meta = {"config": "rmat20", "blocks": [], "total_products": int(per.sum()), "group": GROUP}
    arrays = {}
    rng = np.random.default_rng(3)
    for i, (lo, hi) in enumerate(blocks):
        sub = matgen.rows_slice(a, lo, hi)
        t0 = time.perf_counter()
        c, rep = sg.spgemm(ref_csr(sub), bref, sg.EngineConfig(workers=os.cpu_count() or 1, seed=0,
                                                                workflow=sg.WorkflowOverride.FORCE_SYMBOLIC))
        dt = time.perf_counter() - t0
        p = pin(c, rng, nsample=4)
        m = p["meta"]
        m.update({"lo": lo, "hi": hi, "products": int(per[lo:hi].sum()), "reference_seconds": dt})
        meta["blocks"].append(m)
        for k, v in p["arrays"].items():
            arrays[f"b{i}_{k}"] = v
        print(f"rmat20 block {i} rows [{lo},{hi}) products {m['products']} nnz {m['nnz']} {dt:.1f}s", flush=True)
    save("rmat20_blocks", meta, arrays)


def main():
    which = sys.argv[1:] or ["poisson64", "rect", "rmat20"]
    for w in which:
        if w == "rmat20":
            rmat20_blocks()
        else:
            whole(w)


if __name__ == "__main__":
    main()

"""SpGEMM benchmark: GFLOP/s (2 x intermediate products / s) and HBM-roofline
fraction of C = A*A on the R-MAT scale-20 config (BASELINE.json configs[2],
the config the north star's >= 50 % roofline target is quoted on).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config rmat20|poisson64|rect|er10k|rmatNN] [--dtype f64|f32]

One step = one full ``spgemm`` (analysis, sketch/sample, prediction, binning,
numeric, fallback, compaction) over device-resident A and B, producing the
device-resident CSR C.  N > 1: rows of A are sharded across ranks by balanced
intermediate-product count (weak work split of one matrix; no data-path
collective), the max over ranks is timed.  ``--impl reference`` times the
reference algorithm's CPU restatement (oracle/ocean_cpu.py, the reference's
own numpy path) on a bounded products-balanced row-block sample, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
from dataclasses import replace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# C of R-MAT-20 is 116 GB: avoid caching-allocator fragmentation between steps
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmat20")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--workflow", default="auto", choices=["auto", "symbolic", "estimate", "upper"],
                    help="WorkflowOverride of every step (estimate = FORCE_ESTIMATE: the HLL-estimate-driven "
                         "workflow, reference engine.py:166-171)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-warmup", type=int, default=1,
                    help="untimed end-to-end calls first (they pin the recycled host result buffers)")
    ap.add_argument("--parity-blocks", type=int, default=8,
                    help="row blocks of matgen.stratified_blocks the reference CPU engine runs (timed as the "
                         "cpu_baseline leg, and compared entry by entry with this run's C)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--batch-products", type=float, default=None,
                    help="N>1: rows of each rank run in batches of at most this many products (default: "
                         "4e9 for R-MAT-23, whose C does not fit in HBM; none otherwise)")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def compulsory_bytes(m, k, nnz_a, products, nnz_c, v):
    """8(m+1) + (4+v) nnz_A + 8(k+1) + (4+v) products + 8(m+1) + (4+v) nnz_C
    (BASELINE.md §2)."""
    return 8 * (m + 1) + (4 + v) * nnz_a + 8 * (k + 1) + (4 + v) * products + 8 * (m + 1) + (4 + v) * nnz_c


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        """Starts the sampler and waits for its first sample, so NVML's
        start-up (which holds driver locks) happens before the timed region."""
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.reader = threading.Thread(target=self._read, daemon=True)
        self.reader.start()
        t0 = time.time()
        while not self.lines and time.time() - t0 < 10 and self.proc.poll() is None:
            time.sleep(0.01)
        self.skip = len(self.lines)  # samples taken before the timed region

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.reader.join(timeout=5)
        out = "".join(self.lines[max(self.skip - 1, 0):])
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class CpuReference:
    """The reference's own CPU engine, timed on this host's cores.

    ``baseline/_ref`` holds the unmodified reference package
    (``pip install --target baseline/_ref /root/reference/pkg``, see
    DESIGN.md); it is imported from there (kind "reference").  When it is
    absent the oracle port of the same engine is used (kind "port").

    R-MAT-20's whole product needs ~0.9 TB of host memory in the reference,
    so the full-matrix time is extrapolated from row blocks
    (``matgen.stratified_blocks``; rows are independent, engine.py:13-14):
    the per-call fixed cost -- row statistics over all of A, B's sketches,
    the sampled CR and the workflow choice (engine.py:147-174) -- is timed
    once on the whole matrix, and every block runs the rest of the pipeline
    (predict .. compact, engine.py:177-216) with the whole matrix's workflow
    forced, so  T_full = T_fixed + sum(T_block) * total / sum(products_block).
    """

    def __init__(self, workers):
        self.workers = workers
        path = os.path.join(ROOT, "baseline", "_ref")
        self.sg = None
        if os.path.isdir(os.path.join(path, "sketchgemm")):
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                import sketchgemm
                self.sg = sketchgemm
            except Exception:  # reported as kind "port"
                self.sg = None
        self.kind = "reference" if self.sg is not None else "port"
        if self.sg is None:
            from oracle import ocean_cpu
            self.oc = ocean_cpu

    def _csr(self, m):
        if self.sg is None:
            return m
        return self.sg.CsrMatrix(m.nrows, m.ncols, np.asarray(m.row_ptr), np.asarray(m.col_idx),
                                 np.asarray(m.values))

    def fixed(self, a, b):
        """(seconds, workflow) of the per-call stages on the whole matrix."""
        t0 = time.perf_counter()
        if self.sg is not None:
            from sketchgemm import analysis as an
            A, B = self._csr(a), self._csr(b)
            st = an.compute_row_stats(A, B)
            avg = st.avg_products()
            regs = an.select_registers(st.er)
            if avg < 64:
                wf = "upper"
            else:
                sk = an.build_b_sketches(B, {32: 5, 64: 6, 128: 7}[regs])
                smp = an.sample_cr(A, sk, st, 0.03, 600, 10_000, 0)
                wf = an.select_workflow(avg, st.er, smp.cr_hat).value  # "symbolic" / "estimate" / "upper"
        else:
            oc = self.oc
            st = oc.row_stats(a, b)
            avg = st.total / a.nrows if a.nrows else 0.0
            regs = oc.choose_registers(st.er)
            if avg < 64:
                wf = "upper"
            else:
                sk = oc.b_sketches(b, oc.P_OF_M[regs])
                rows = oc.sample_rows(a.nrows, oc.SAMPLE_RATIO, oc.SAMPLE_MIN, oc.SAMPLE_MAX, 0)
                cr = oc.cr_from_sample(st.products[rows], oc.merged_estimates(a, sk, rows))
                wf = oc.choose_workflow(avg, st.er, cr[0])
        return time.perf_counter() - t0, wf

    def whole(self, a, b):
        """AUTO on the whole matrix: (C, seconds)."""
        if self.sg is not None:
            return self.sg.spgemm(self._csr(a), self._csr(b), self.sg.EngineConfig(workers=self.workers, seed=0))
        return self.oc.spgemm(a, b, workers=self.workers)

    def block(self, a, b, lo, hi, wf):
        """(C rows [lo, hi) as host CSR, seconds of the non-fixed stages)."""
        from paper_2604_19004_b200.matgen import rows_slice
        sub = rows_slice(a, lo, hi)
        if self.sg is not None:
            ov = {"symbolic": self.sg.WorkflowOverride.FORCE_SYMBOLIC,
                  "estimate": self.sg.WorkflowOverride.FORCE_ESTIMATE,
                  "upper": self.sg.WorkflowOverride.FORCE_UPPER_BOUND}[wf]
            c, rep = self.sg.spgemm(self._csr(sub), self._csr(b),
                                    self.sg.EngineConfig(workers=self.workers, seed=0, workflow=ov))
            ms = rep.total_ms - rep.analysis_ms - rep.sketch_ms
        else:
            c, rep = self.oc.spgemm(sub, b, workflow=wf, workers=self.workers)
            ms = rep["total_ms"] - rep["analysis_ms"] - rep["sketch_ms"]
        return c, ms / 1e3


WHOLE_MAX_PRODUCTS = 4e8  # configs up to this size run whole in the reference


def cpu_baseline(a, b, workers, nblocks=None, budget_s=None, warmup=0, keep=False):
    """Time the reference CPU engine on this config.

    Configs of at most WHOLE_MAX_PRODUCTS products run whole (ER-10k,
    Poisson 64^3, rect: BASELINE.md §3).  Larger ones run the blocks of
    ``matgen.stratified_blocks`` in list order -- `warmup` untimed blocks
    first, then timed blocks until `nblocks` are done or `budget_s` is spent
    (at least one) -- and extrapolate (see CpuReference).  Returns a dict with
    GFLOP/s and the sample description; the blocks' C when keep=True."""
    from paper_2604_19004_b200 import matgen
    ref = CpuReference(workers)
    per = matgen.row_products(a, b)
    total = int(per.sum())
    if total <= WHOLE_MAX_PRODUCTS:
        secs, outs = [], []
        for i in range(min(warmup, 1) + max(1, min(nblocks or 3, 3))):
            t0 = time.perf_counter()
            c, _ = ref.whole(a, b)
            if i >= min(warmup, 1):
                secs.append(time.perf_counter() - t0)
                if keep and not outs:
                    outs.append(c)
        t = float(np.mean(secs))
        return {"value": 2.0 * total / t / 1e9, "unit": "GFLOP/s", "cores": workers, "kind": ref.kind,
                "sample": f"whole matrix, AUTO workflow, mean of {len(secs)} calls ({t:.2f} s each)",
                "extrapolated_seconds": t, "blocks": [(0, a.nrows)], "outputs": outs, "total_products": total}
    blocks = matgen.stratified_blocks(per)
    t_fixed, wf = ref.fixed(a, b)
    for i in range(warmup):
        lo, hi = blocks[i % len(blocks)]
        ref.block(a, b, lo, hi, wf)
    done, t_var, used, outs = 0, 0.0, [], []
    t_start = time.perf_counter()
    for j in range(nblocks if nblocks is not None else len(blocks)):
        if budget_s is not None and used and time.perf_counter() - t_start > budget_s:
            break
        lo, hi = blocks[j % len(blocks)]
        c, sec = ref.block(a, b, lo, hi, wf)
        t_var += sec
        done += int(per[lo:hi].sum())
        used.append((lo, hi))
        if keep:
            outs.append(c)
    t_full = t_fixed + t_var * total / max(done, 1)
    uniq = sorted(set(used))
    cover = sum(int(per[lo:hi].sum()) for lo, hi in uniq)
    desc = (f"{len(used)} timed row blocks ({len(uniq)} distinct) of matgen.stratified_blocks, rows "
            + ", ".join(f"[{lo},{hi})" for lo, hi in uniq[:5]) + (", ..." if len(uniq) > 5 else "")
            + f"; {cover} distinct products = {100.0 * cover / max(total, 1):.3f}% of all {total}; "
            f"{wf} workflow forced as AUTO picks on the whole matrix; fixed per-call stages (row stats, "
            f"B sketches, sampled CR: engine.py:147-174) {t_fixed:.2f} s timed once on the whole matrix; "
            f"full time = fixed + block time x total / sampled products = {t_full:.1f} s")
    return {"value": 2.0 * total / t_full / 1e9, "unit": "GFLOP/s", "cores": workers, "kind": ref.kind,
            "sample": desc, "workflow": wf, "fixed_seconds": t_fixed, "block_seconds": t_var,
            "extrapolated_seconds": t_full, "blocks": used, "outputs": outs, "total_products": total}


def parity_rows(a, b, c, nblocks):
    """Host copies of the rows of device C that the parity check compares:
    the first `nblocks` stratified blocks (the whole C for configs that the
    reference runs whole), plus the 5 rows around the 2^31 output offset."""
    from paper_2604_19004_b200 import matgen
    per = matgen.row_products(a, b)
    if int(per.sum()) <= WHOLE_MAX_PRODUCTS:
        blocks = [(0, a.nrows)]
    else:
        blocks = matgen.stratified_blocks(per)[:nblocks]
    out = {blk: c.rows(*blk) for blk in blocks}
    rp = c.row_ptr
    if int(rp[-1]) > 2 ** 31:
        import torch
        r = int(torch.searchsorted(rp, torch.tensor([2 ** 31], dtype=torch.int64, device=rp.device),
                                   right=True)[0]) - 1
        blk = (max(0, r - 2), min(a.nrows, r + 3))
        out[blk] = c.rows(*blk)
    return out


def check_parity(a, b, rows, cb):
    """Entry-by-entry comparison of this run's C rows with the reference CPU
    engine's output for the same rows (the reference comparator,
    pkg/tests/matgen.py:151-156: structure exact, values rtol 1e-12, atol 0)."""
    ref = dict(zip(cb["blocks"], cb["outputs"]))
    extra = [blk for blk in rows if blk not in ref]
    if extra:
        cr = CpuReference(cb["cores"])
        for lo, hi in extra:
            ref[(lo, hi)], _ = cr.block(a, b, lo, hi, cb.get("workflow", "symbolic"))
    nrows = ok_struct = 0
    worst = 0.0
    bad = []
    for blk, mine in rows.items():
        r = ref[blk]
        same = (np.array_equal(np.asarray(mine.row_ptr), np.asarray(r.row_ptr))
                and np.array_equal(np.asarray(mine.col_idx), np.asarray(r.col_idx)))
        nrows += blk[1] - blk[0]
        if not same:
            bad.append(list(blk))
            continue
        ok_struct += 1
        rv = np.asarray(r.values, dtype=np.float64)
        if len(rv):
            worst = max(worst, float(np.max(np.abs(np.asarray(mine.values, dtype=np.float64) - rv) / np.abs(rv))))
    return {"blocks": len(rows), "rows": int(nrows), "structure_equal_blocks": ok_struct,
            "max_rel_err": worst, "ok": not bad and worst <= 1e-12, "mismatched_blocks": bad,
            "against": f"{cb['kind']} CPU engine on the same rows (structure exact, values rtol 1e-12)",
            "row_blocks": [list(x) for x in rows]}


TIMED_KERNELS = ("k_win", "k_bmr", "k_win_light", "k_hash_warp", "k_hash_block", "k_bitmap",
                 "k_hash_warp:count", "k_hash_block:count", "k_bitmap:count")


def kernel_times(lib):
    """Event-timed totals of the dominant kernels (sg_kernel_time)."""
    out = {}
    for k in TIMED_KERNELS:
        ms = ctypes.c_double(0.0)
        n = ctypes.c_int64(0)
        if lib.sg_kernel_time(k.encode(), ctypes.byref(ms), ctypes.byref(n)) == 0 and n.value:
            out[k] = (ms.value, n.value)
    return out


def ncu_traffic(config, kernel, brackets_per_step=1):
    """DRAM bytes of `kernel` per timed bracket, from the committed ncu launch
    list of one step of the same command (a bracket may span several launches,
    e.g. the two window-kernel classes)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)[config][kernel]
        return d.get("dram_bytes_per_step", d["dram_bytes_per_launch"] * d["launches"]) / max(brackets_per_step, 1)
    except (OSError, KeyError, ValueError):
        return None


def ncu_dominant(config):
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)[config]
        return max(d, key=lambda k: d[k].get("us_per_step", d[k]["us_per_launch"] * d[k]["launches"]))
    except (OSError, KeyError, ValueError):
        return None


def make_inputs(name):
    from paper_2604_19004_b200 import matgen
    return matgen.make_config(name)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = max(world, 1)
    workload = {"rmat20": "C=A*A R-MAT scale 20 edge-factor 16 (BASELINE configs[2])",
                "poisson64": "C=A*A 27-point Poisson 64^3 (configs[1])",
                "rect": "C=A*B 1M x 64k * 64k x 1M, 16/row (configs[3])",
                "er10k": "C=A*A Erdos-Renyi 10k, 8/row (configs[0])"}.get(args.config, f"C=A*A {args.config}")
    metric = "SpGEMM GFLOP/s (2 x intermediate products / s)"

    if args.impl == "reference":
        if rank != 0:
            return
        a, b = make_inputs(args.config)
        workers = os.cpu_count() or 1
        cb = cpu_baseline(a, b, workers, nblocks=args.steps, warmup=args.warmup)
        v = cb["value"]
        line = {"metric": metric, "value": v, "unit": "GFLOP/s", "n_gpus": n_gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": cb["extrapolated_seconds"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator, SURVEY §8d; values U[0.5,1.5])",
                "impl": "reference",
                "config": {"workload": workload, "m": a.nrows, "k": b.nrows, "n": b.ncols, "nnz_a": a.nnz,
                           "products": cb.get("total_products"), "parallelism": f"cpu threads x{workers}",
                           "workflow": cb.get("workflow")},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2604_19004_b200 import EngineConfig, _lib, spgemm
    from paper_2604_19004_b200.device import DeviceCsr, to_device

    # test hooks for the N>1 path on a one-GPU box: every rank on cuda:0 over gloo
    same_dev = os.environ.get("SG_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        backend = os.environ.get("SG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's own log shows the communicator (nranks, NVLS / NVLink
            # transport) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    lib = _lib.load()
    # the root builds the inputs; under torchrun the other ranks receive them
    # over NCCL (plan_shards), so they skip the host generation
    a, b = make_inputs(args.config) if (world == 1 or rank == 0) else (None, None)
    same = b is a
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    vbytes = 8 if args.dtype == "f64" else 4
    from paper_2604_19004_b200 import WorkflowOverride
    wf_over = WorkflowOverride(args.workflow)
    cfg = EngineConfig(return_device=True, dtype=args.dtype, workflow=wf_over)
    if n_gpus == 1:
        a_loc = a
        A = to_device(a, dev, dt)
        B = A if same else to_device(b, dev, dt)

        def step():
            return spgemm(A, B, cfg)
    else:
        # row-sharded job (shard.py), planned ONCE outside the timed loop:
        # B (= A) broadcast from rank 0 over NCCL, A's rows cut by balanced
        # products (row-stats kernel on rank 0), the workflow decided once
        # for the whole product on rank 0 and broadcast.  A step multiplies
        # the local rows (in product-bounded batches when C does not fit the
        # GPU: R-MAT-23) and exchanges nnz offsets; no data-path collective.
        from paper_2604_19004_b200.shard import (gpu_decide_fn, gpu_local_fn, gpu_products_fn, plan_shards,
                                                 run_shard)
        A0 = to_device(a, dev, dt) if rank == 0 else None
        B0 = (A0 if same else to_device(b, dev, dt)) if rank == 0 else None
        # (only the root holds the inputs: it decides whether rows are batched)
        big = [a is not None and a.nnz > 50_000_000]
        dist.broadcast_object_list(big, src=0)
        budget = args.batch_products or (4e9 if big[0] else None)
        plan = plan_shards(A0, B0, device=dev, products_fn=gpu_products_fn(dev),
                           decide_fn=gpu_decide_fn(cfg, dev), batch_products=budget)
        del A0, B0
        local_fn = gpu_local_fn(cfg)
        checks = torch.zeros(2, dtype=torch.float64, device=dev)

        def consume(lo, hi, rp, ci, vv):
            # C batches that do not stay resident leave a checksum
            checks[0] += vv.double().sum()
            checks[1] += ci.double().sum()

        def step():
            sh = run_shard(plan, local_fn, consume=consume if len(plan.batches) > 1 else None)
            return sh, sh.report

        a_loc = None
    torch.cuda.synchronize()

    c = rep = None
    for _ in range(args.warmup):
        c, rep = step()
        del c
    stream = torch.cuda.current_stream(dev)
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    lib.sg_kernel_timer(1)
    l0 = lib.sg_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    stage_ms = {}
    nnz_c_loc = 0
    prod_loc = 0
    for _ in range(args.steps):
        c, rep = step()
        for k, v in (rep.kernel_ms or {}).items():
            stage_ms[k] = stage_ms.get(k, 0.0) + v
        nnz_c_loc = rep.nnz_c
        prod_loc = rep.total_products
        c_last_local = getattr(c, "local", None)
        if _ < args.steps - 1:
            del c
    e1.record(stream)
    torch.cuda.synchronize()
    launches = int(lib.sg_launch_count() - l0)
    ktimes = kernel_times(lib)
    lib.sg_kernel_timer(0)
    # rows of the last timed step's C kept for the parity check against the
    # reference CPU engine (cpu_baseline leg below): the parity row blocks
    # plus the rows whose output offsets cross 2^31 (int64 offsets)
    check_rows = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu:
        check_rows = parity_rows(a, b, c, args.parity_blocks)
    del c
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, nnz_c_loc, prod_loc], dtype=torch.float64, device=dev)
    if world > 1:
        # the stitched report already holds whole-product nnz_c / products
        # (run_shard sums them over ranks); time is the max over ranks
        dist.all_reduce(t[0:1], op=dist.ReduceOp.MAX)
        nnz_c_loc, prod_loc = c_last_local["nnz_c"], c_last_local["products"]
    ms_tot, nnz_c, products = float(t[0]), int(t[1]), int(t[2])
    ms_step = ms_tot / args.steps
    gflops = 2.0 * products / (ms_step * 1e-3) / 1e9

    # roofline of the dominant stage on this rank (CUDA events on the launch stream)
    peak, peak_kind = load_peaks()
    m, k = (a.nrows, b.nrows) if a is not None else (plan.A[0], plan.B[0])
    loc_rows = a_loc.nrows if a_loc is not None else c_last_local["rows"]
    loc_nnz = a_loc.nnz if a_loc is not None else c_last_local["nnz_a"]
    alg = compulsory_bytes(loc_rows, k, loc_nnz, prod_loc, nnz_c_loc, vbytes)
    per_step = {kk: v / args.steps for kk, v in stage_ms.items() if kk != "h2d"}
    dom = max(per_step, key=per_step.get) if per_step else "numeric"
    num_ms = per_step.get("numeric", 0.0) + per_step.get("fallback", 0.0) + per_step.get("compact", 0.0)
    achieved = alg / (num_ms * 1e-3) / 1e9 if num_ms > 0 else None
    step_gbs = alg / (ms_step * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": "numeric+fallback+compact stages (Gustavson pass)",
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": None,
            "algorithmic_bytes_per_step": alg, "dominant_stage": dom}
    # dominant kernel: largest share of the committed ncu launch list of this
    # config (the bin kernels run concurrently on side streams, so their
    # event brackets overlap and cannot rank them); else the event timers
    dk = ncu_dominant(args.config)
    if dk not in ktimes:
        dk = max(ktimes, key=lambda kk: ktimes[kk][0]) if ktimes else None
    if dk in ("k_win", "k_bmr") and n_gpus == 1:
        # the window kernel: algorithmic bytes of the rows it processes (one
        # extra untimed call collects their totals), over its event-timed
        # average launch duration
        c_ws, rs = spgemm(A, B, replace(cfg, window_stats=True))
        del c_ws  # C is >100 GB at R-MAT-20: free it before the e2e run
        ws_ = rs.window_stats
        # k_win writes both halves of the windows' C entries (columns from
        # its bitmap, values); k_bmr with saved bitmaps only the values
        cbytes = (4 + vbytes) if (dk == "k_win" or not ws_["saved_bitmaps"]) else vbytes
        kb = (16 * ws_["rows"] + (4 + vbytes) * ws_["nnz_a"] + (4 + vbytes) * ws_["products"]
              + cbytes * ws_["nnz_c"])
        kms_, kn_ = ktimes[dk]
        ach = kb / (kms_ / kn_ * 1e-3) / 1e9
        traffic = ncu_traffic(args.config, dk, kn_ / args.steps)
        roof = {"bound": "hbm", "kernel": dk, "achieved": ach, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": kb, "ms_per_launch": kms_ / kn_,
                "share_of_step": kms_ / ms_tot,
                "units_per_launch": {kk: ws_[kk] for kk in ("rows", "windows", "nnz_a", "products", "nnz_c")},
                "bytes_per_unit": f"16/row + {4 + vbytes}/A entry + {4 + vbytes}/product + {cbytes}/C entry",
                "traffic_source": "profiles/ncu_traffic.json (ncu launch list of the same command)",
                "whole_pass": {"achieved": achieved, "frac": (achieved / peak) if achieved else None,
                               "algorithmic_bytes_per_step": alg}}
    elif dk is not None:
        roof["traffic"] = ncu_traffic(args.config, dk)
        roof["dominant_kernel"] = dk
        roof["traffic_source"] = "profiles/ncu_traffic.json (dominant kernel, per launch)"
    # the whole multiply against the same HBM roof (algorithmic bytes / step time)
    roof["whole_step"] = {"achieved": step_gbs, "frac": step_gbs / peak, "algorithmic_bytes_per_step": alg}
    roof["kernel_ms_per_step"] = {kk: round(v[0] / args.steps, 3) for kk, v in ktimes.items()}
    roof["kernel_ms_note"] = ("CUDA-event brackets on the launching stream; bin kernels (k_hash_*, k_bitmap) "
                              "run concurrently on side streams, so their brackets overlap")

    # e2e through the public API with host buffers (H2D + D2H inside the timed region)
    e2e = None
    torch.cuda.empty_cache()
    if not args.no_e2e and n_gpus > 1 and len(plan.batches) > 1:
        e2e = {"value": None, "unit": "GFLOP/s",
               "skipped": "C does not fit in host memory (R-MAT-23: ~2 TB); batches are checksummed on device"}
    elif not args.no_e2e:
        try:
            cfg_h = EngineConfig(dtype=args.dtype, host_pool=True, workflow=wf_over)
            a_h = a if (a is None or args.dtype == "f64") else a.astype(np.float32)
            b_h = (a_h if same else (b if (b is None or args.dtype == "f64") else b.astype(np.float32)))
            ts = []
            cbytes = 0
            from paper_2604_19004_b200.device import HOST_POOL
            for it in range(args.e2e_warmup + max(1, args.e2e_steps)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if n_gpus == 1:
                    ch, rh = spgemm(a_h, b_h, cfg_h)
                    cbytes = ch.row_ptr.nbytes + ch.col_idx.nbytes + ch.values.nbytes
                else:
                    from paper_2604_19004_b200.device import download
                    from paper_2604_19004_b200.shard import gpu_local_fn, gpu_products_fn, spgemm_sharded
                    from paper_2604_19004_b200.shard import gpu_decide_fn
                    sh = spgemm_sharded(a_h if rank == 0 else None, b_h if rank == 0 else None,
                                        gpu_local_fn(cfg), device=dev, gather=False,
                                        products_fn=gpu_products_fn(dev), decide_fn=gpu_decide_fn(cfg, dev))
                    ch = [download(sh.row_ptr, pool=HOST_POOL), download(sh.col_idx, pool=HOST_POOL),
                          download(sh.values, pool=HOST_POOL)]
                    cbytes = sum(x.nbytes for x in ch)
                torch.cuda.synchronize()
                if it >= args.e2e_warmup:
                    ts.append(time.perf_counter() - t0)
                del ch
            h2d = (a_h.row_ptr.nbytes + a_h.col_idx.nbytes + a_h.values.nbytes) if a_h is not None else 0
            if b_h is not a_h and b_h is not None:
                h2d += b_h.row_ptr.nbytes + b_h.col_idx.nbytes + b_h.values.nbytes
            if n_gpus > 1 and rank != 0:
                h2d = 0  # only the root uploads; the others receive over NVLink
            tw = torch.tensor([max(ts) if world > 1 else float(np.mean(ts))], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tw, op=dist.ReduceOp.MAX)
            e2e = {"value": 2.0 * products / float(tw[0]) / 1e9, "unit": "GFLOP/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(cbytes),
                   "seconds_per_step": float(tw[0]), "steps": len(ts), "warmup": args.e2e_warmup,
                   "host": "host CsrMatrix in; C downloaded into recycled pinned host buffers "
                           "(EngineConfig(host_pool=True)), one DMA per 256 MB chunk"}
        except Exception as exc:  # reported in the JSON line, never dropped silently
            e2e = {"value": None, "unit": "GFLOP/s", "error": f"{type(exc).__name__}: {exc}"[:300]}

    cpu = parity = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu:
        cb = cpu_baseline(a, b, os.cpu_count() or 1, nblocks=args.parity_blocks, keep=True)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        parity = check_parity(a, b, check_rows, cb)

    if rank == 0:
        line = {
            "metric": metric, "value": gflops, "unit": "GFLOP/s", "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if n_gpus > 1 else "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded generator, SURVEY §8d; values U[0.5,1.5])",
            "config": {"workload": workload, "m": m, "k": k, "n": b.ncols, "nnz_a": a.nnz,
                       "products": products, "nnz_c": nnz_c, "parallelism": f"row-shard x{n_gpus}",
                       "l2": "no flush needed: every step writes C (>> 126 MB L2)",
                       "workflow": rep.workflow if rep else None,
                       "workflow_override": args.workflow,
                       "stage_ms": {kk: round(v, 3) for kk, v in per_step.items()},
                       "shard_rank0": c_last_local if n_gpus > 1 else None,
                       "c_checksum": ([float(x) for x in checks.tolist()] if (n_gpus > 1 and len(plan.batches) > 1)
                                      else None),
                       # north star: sketch + sampled CR + (estimate workflow) all-row estimate,
                       # as a share of the whole step
                       "estimation_share": ((per_step.get("sketch", 0.0)
                                             + (per_step.get("predict", 0.0) if rep and rep.workflow == "estimate"
                                                else 0.0)) / ms_step) if ms_step else None,
                       "hbm_frac_whole_step": step_gbs / peak},
            "roofline": roof,
            "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

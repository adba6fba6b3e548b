"""The row-sharded path with the GPU engine per rank (shard.gpu_local_fn,
shard.gpu_products_fn) at world size 2.  The box has one GPU, so both ranks
share cuda:0 and talk over gloo (NCCL refuses two ranks on one device); the
data path -- device broadcast of B, row-stats partition, per-rank engine,
offset exchange, gather -- is the one bench.py runs over NCCL."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from test_shard_gloo import _free_port

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, case, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(rank, case, out_q)
    except Exception as exc:  # surface worker failures to the parent
        import traceback
        out_q.put(("error", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run(rank, case, out_q):
    if case.startswith("batched:"):
        return _run_batched(rank, case.split(":", 1)[1], out_q)
    if True:
        from golden_io import Case
        from paper_2604_19004_b200 import EngineConfig
        from paper_2604_19004_b200.device import to_device
        from paper_2604_19004_b200.shard import gpu_local_fn, gpu_products_fn, spgemm_sharded
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        c = Case(case)
        a = to_device(c.A, dev) if rank == 0 else None
        b = to_device(c.B, dev) if rank == 0 else None
        shard = spgemm_sharded(a, b, gpu_local_fn(EngineConfig()), device=dev, gather=True,
                               products_fn=gpu_products_fn(dev))
        if rank == 0:
            out_q.put((shard.row_ptr.cpu().numpy(), shard.col_idx.cpu().numpy(), shard.values.cpu().numpy()))
        else:
            out_q.put(("rank1", shard.row_lo, shard.row_hi))


@pytest.mark.parametrize("case", ["pair05", "corpus2"])
def test_gpu_sharded_equals_reference(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from golden_io import Case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(2)]
    errs = [g for g in got if isinstance(g[0], str) and g[0] == "error"]
    assert not errs, errs[0][2]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = [g for g in got if not isinstance(g[0], str)][0]
    c = Case(case)

    class C:
        nrows, ncols = c.A.nrows, c.B.ncols
        row_ptr, col_idx, values = full
    c.check_product(C)
    np.testing.assert_array_equal(full[0][-1:], [c.d["C_ptr"][-1]])


def _run_batched(rank, case, out_q):
    """plan_shards with the root's GPU decision and product-bounded batches;
    two steps reuse one plan; batches stream through `consume`."""
    from golden_io import Case
    from paper_2604_19004_b200 import EngineConfig
    from paper_2604_19004_b200.device import to_device
    from paper_2604_19004_b200.shard import gpu_decide_fn, gpu_local_fn, gpu_products_fn, plan_shards, run_shard
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    c = Case(case)
    a = to_device(c.A, dev) if rank == 0 else None
    b = to_device(c.B, dev) if rank == 0 else None
    cfg = EngineConfig()
    budget = max(1, int(c.d["products"].sum()) // 9)
    plan = plan_shards(a, b, device=dev, products_fn=gpu_products_fn(dev), decide_fn=gpu_decide_fn(cfg, dev),
                       batch_products=budget)
    got = {}

    def consume(lo, hi, rp, ci, vv):
        got[(lo, hi)] = (rp.cpu().numpy(), ci.cpu().numpy(), vv.cpu().numpy())
    for _ in range(2):
        got.clear()
        sh = run_shard(plan, gpu_local_fn(cfg), consume=consume)
    r = sh.report
    out_q.put((rank, len(plan.batches), got, {k: getattr(r, k) for k in
                                              ("workflow", "registers", "er", "cr_hat", "nnz_c",
                                               "overflow_row_count", "total_products", "bitmap_query")}))


@pytest.mark.parametrize("case", ["corpus1", "enhanced"])
def test_gpu_sharded_batched_with_global_decision(case):
    """Config-5 machinery on one GPU (two ranks, gloo): whole-product
    decision on the root, batches through consume, stitched report equal to
    the reference's whole-product report, batches equal to the reference C."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from golden_io import Case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "batched:" + case, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    errs = [g for g in got if isinstance(g[0], str) and g[0] == "error"]
    assert not errs, errs[0][2]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = Case(case)
    want = c.meta["reports"]["auto"]
    cp, cc, cv = c.d["C_ptr"], c.d["C_col"], c.d["C_val"]
    nb = 0
    for rank, nbatch, batches, rep in got:
        nb += nbatch
        for k in ("workflow", "registers", "nnz_c", "overflow_row_count", "total_products", "bitmap_query"):
            assert rep[k] == want[k], (rank, k, rep[k], want[k])
        assert rep["er"] == pytest.approx(want["er"], rel=1e-12)
        assert rep["cr_hat"] == pytest.approx(want["cr_hat"], rel=1e-12)
        for (lo, hi), (rp, ci, vv) in batches.items():
            np.testing.assert_array_equal(rp, cp[lo:hi + 1] - cp[lo])
            np.testing.assert_array_equal(ci, cc[cp[lo]:cp[hi]])
            if c.stride == 1:
                np.testing.assert_allclose(vv, cv[cp[lo]:cp[hi]], rtol=1e-12, atol=0)
    assert nb > 2


def test_bench_torchrun_two_ranks_one_gpu():
    """The driver's multi-GPU bench launch (torchrun, rank 0 alone holds the
    inputs), both arms, with two ranks on cuda:0 over gloo."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SG_BENCH_SAME_DEVICE="1", SG_BENCH_BACKEND="gloo")
    for extra in ([], ["--impl", "reference"]):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
               "--config", "rmat12", "--steps", "2", "--warmup", "3", "--no-e2e"] + extra
        r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert line["n_gpus"] == 2 and line["value"] > 0
        if not extra:
            assert line["config"]["nnz_c"] > 0

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

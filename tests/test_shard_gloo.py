"""Multi-process (world size 2, gloo, CPU) tests of the row-sharded path's
host logic: balanced partition, broadcast of B, offset exchange, stitching.
The per-rank multiply is the oracle here (test-only); on GPUs it is the
engine (shard.gpu_local_fn) over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_local_fn(nrows, ncols_a, row_ptr, col_idx, values, B):
    from oracle import ocean_cpu as oc
    a = oc.Csr(nrows, ncols_a, row_ptr.numpy(), col_idx.numpy(), values.numpy())
    b = oc.Csr(B[0], B[1], B[2].numpy(), B[3].numpy(), B[4].numpy())
    c, rep = oc.spgemm(a, b)
    return (torch.from_numpy(c.row_ptr), torch.from_numpy(c.col_idx), torch.from_numpy(c.values), rep)


def _worker(rank, world, port, case, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from golden_io import Case
        from paper_2604_19004_b200.shard import spgemm_sharded
        c = Case(case)
        a = c.A if rank == 0 else None
        b = c.B if rank == 0 else None
        if case == "cfg1_er10k" and rank == 0:
            b = a  # A*A shares one broadcast
        shard = spgemm_sharded(a, b, oracle_local_fn, gather=True)
        if rank == 0:
            out_q.put((shard.row_ptr.numpy(), shard.col_idx.numpy(), shard.values.numpy()))
        else:
            out_q.put(("rank1", shard.row_lo, shard.row_hi, shard.nnz_offset, shard.nnz_total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["pair00", "corpus1", "cfg1_er10k"])
def test_sharded_gather_equals_reference(case):
    from golden_io import Case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = [o for o in outs if not (isinstance(o[0], str))][0]
    r1 = [o for o in outs if isinstance(o[0], str)][0]
    c = Case(case)
    from paper_2604_19004_b200.csr import CsrMatrix
    C = CsrMatrix(c.A.nrows, c.B.ncols, full[0], full[1], full[2])
    c.check_product(C)
    # rank 1's shard starts where rank 0's rows end, offsets stitch exactly
    _, lo, hi, off, total = r1
    assert hi == c.A.nrows and total == int(c.d["C_ptr"][-1])
    assert off == int(c.d["C_ptr"][lo])


def test_balanced_cuts_properties():
    from paper_2604_19004_b200.shard import balanced_cuts
    rng = np.random.default_rng(0)
    for parts in (1, 2, 4, 8):
        per = rng.pareto(1.2, 10_000).astype(np.int64) * 100
        cuts = balanced_cuts(per, parts)
        assert cuts[0] == 0 and cuts[-1] == len(per) and cuts == sorted(cuts)
        sums = [per[cuts[i]:cuts[i + 1]].sum() for i in range(parts)]
        assert max(sums) <= per.sum() / parts + per.max()
    assert balanced_cuts(np.zeros(5, np.int64), 3)[-1] == 5


def oracle_decide_fn(A, B):
    """decide_fn for the CPU ranks: the oracle's analysis + sample stages on
    the whole operands (engine.py:147-174)."""
    from oracle import ocean_cpu as oc
    from paper_2604_19004_b200.engine import Decision
    a = oc.Csr(A.nrows, A.ncols, A.row_ptr.numpy(), A.col_idx.numpy(), A.values.numpy())
    b = oc.Csr(B.nrows, B.ncols, B.row_ptr.numpy(), B.col_idx.numpy(), B.values.numpy())
    st = oc.row_stats(a, b)
    avg = st.total / a.nrows if a.nrows else 0.0
    regs = oc.choose_registers(st.er)
    if avg < 64:
        return Decision("upper", regs, st.er, None, st.total)
    sk = oc.b_sketches(b, oc.P_OF_M[regs])
    rows = oc.sample_rows(a.nrows, oc.SAMPLE_RATIO, oc.SAMPLE_MIN, oc.SAMPLE_MAX, 0)
    cr = oc.cr_from_sample(st.products[rows], oc.merged_estimates(a, sk, rows))
    return Decision(oc.choose_workflow(avg, st.er, cr[0]), regs, st.er, tuple(cr), st.total)


def oracle_local_fn_decided(nrows, ncols_a, row_ptr, col_idx, values, B, decision=None):
    from oracle import ocean_cpu as oc
    a = oc.Csr(nrows, ncols_a, row_ptr.numpy(), col_idx.numpy(), values.numpy())
    b = oc.Csr(B[0], B[1], B[2].numpy(), B[3].numpy(), B[4].numpy())
    c, rep = oc.spgemm(a, b, workflow=decision.workflow, registers=decision.registers)
    rep["er"], rep["cr_hat"] = decision.er, (decision.cr[0] if decision.cr else None)
    return (torch.from_numpy(c.row_ptr), torch.from_numpy(c.col_idx), torch.from_numpy(c.values), rep)


def _worker_plan(rank, world, port, case, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from golden_io import Case
        from paper_2604_19004_b200.shard import plan_shards, run_shard
        c = Case(case)
        a = c.A if rank == 0 else None
        b = c.B if rank == 0 else None
        plan = plan_shards(a, b, decide_fn=oracle_decide_fn, batch_products=max(1, int(c.d["products"].sum()) // 7))
        # every step reuses the plan; batches stream through `consume`
        got = {}

        def consume(lo, hi, rp, ci, vv):
            got[(lo, hi)] = (rp.numpy().copy(), ci.numpy().copy(), vv.numpy().copy())
        for _ in range(2):
            got.clear()
            sh = run_shard(plan, oracle_local_fn_decided, consume=consume)
        rep = sh.report
        out_q.put((rank, len(plan.batches), sorted(got), {k: got[k] for k in got},
                   {k: rep[k] for k in ("workflow", "registers", "er", "cr_hat", "nnz_c", "overflow_row_count",
                                        "total_products")}, sh.nnz_offset, sh.nnz_total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["pair03", "corpus0"])
def test_plan_decision_batches_and_report(case):
    """plan_shards/run_shard: the root's whole-product decision reaches every
    rank, rows run in product-bounded batches streamed through `consume`, the
    stitched report counters equal the reference's whole-product report, and
    the batches reassemble the reference C."""
    from golden_io import Case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_plan, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=300) for _ in range(2)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = Case(case)
    want = c.meta["reports"]["auto"]
    cp, cc, cv = c.d["C_ptr"], c.d["C_col"], c.d["C_val"]
    nb = 0
    for rank, nbatch, keys, got, rep, off, total in outs:
        nb += nbatch
        for k in ("workflow", "registers", "nnz_c", "overflow_row_count", "total_products"):
            assert rep[k] == want[k], (rank, k, rep[k], want[k])
        assert rep["er"] == pytest.approx(want["er"], rel=1e-12)
        assert total == int(cp[-1])
        for lo, hi in keys:
            rp, ci, vv = got[(lo, hi)]
            np.testing.assert_array_equal(rp, cp[lo:hi + 1] - cp[lo])
            np.testing.assert_array_equal(ci, cc[cp[lo]:cp[hi]])
            if c.stride == 1:
                np.testing.assert_allclose(vv, cv[cp[lo]:cp[hi]], rtol=1e-12, atol=0)
    assert nb > 2  # the product budget split the ranks' rows into several batches

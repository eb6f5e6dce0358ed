"""DistContext over an NCCL process group on the GPU (world size 1: the only
size one device allows without ranks waiting on one another): group
initialisation, the collective barrier that creates the communicator, the gloo
side group, and the hot path (apply with the overlapped exchange order,
tmmult + compress, ghosted C, mmult) run through that context against the
reference's smoke goldens.  The N > 1 exchanges themselves are covered by the
thread-rank GPU tests and the gloo world-size-2 CPU test."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(port, q):
    import sys
    from pathlib import Path

    import torch
    import torch.distributed as dist

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        from oracle import numpy_oracle as O
        from paper_1907_01005_b200 import _lib
        from paper_1907_01005_b200 import problem as P
        from paper_1907_01005_b200.bcsr import mmult, tmmult
        from paper_1907_01005_b200.comm import DistContext

        _lib.require_device()
        g = dict(np.load(root / "tests" / "golden" / "smoke.npz"))
        ctx = DistContext(device=dev)
        prob = P.build_problem("smoke")
        st = P.make_rank_setup(ctx, prob, device=dev, compact_xc=False)
        st.op.apply(prob.spec_h(), st.x, st.hx)
        tmmult(st.x, st.hx, st.s)
        st.c.update_ghost_values()
        mmult(st.x, st.c, st.xc)
        torch.cuda.synchronize()
        hx = O.per_vector_rel_err(st.hx.to_dense_owned(), g["hx"])
        s = float(np.max(np.abs(st.s.to_dense_owned() - g["s"])) / np.max(np.abs(g["s"])))
        xc = O.per_vector_rel_err(st.xc.to_dense_owned(), g["xc"])
        total = ctx.allreduce_sum(2.5)
        q.put((ctx.backend, ctx.n_ranks, hx, s, xc, total))
    finally:
        dist.destroy_process_group()


def test_nccl_context_runs_the_hot_path(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    p.join(timeout=300)
    if p.is_alive():
        p.kill()
        pytest.fail("NCCL worker hung")
    assert p.exitcode == 0
    backend, n_ranks, hx, s, xc, total = q.get(timeout=10)
    assert backend == "nccl" and n_ranks == 1
    assert hx <= 1e-12 and s <= 1e-11 and xc <= 1e-12, (hx, s, xc)
    assert total == 2.5

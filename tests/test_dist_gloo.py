"""Multi-rank path over torch.distributed (gloo, world size 2, CPU):
layout protocol, ghost update, compress in ascending source order and the
operator's host plan, checked against the reference's 2-rank results."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, degree, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        root = Path(__file__).resolve().parents[1]
        sys.path.insert(0, str(root))
        sys.path.insert(0, str(root / "tests"))
        from _helpers import Small, cosine, emulated_apply

        from paper_1907_01005_b200.comm import DistContext

        g = dict(np.load(root / "tests" / "golden" / "random.npz"))
        ext = tuple(int(v) for v in g[f"p{degree}_extents"])
        s = Small(ext, (1.0, 1.0, 1.0), 1, degree, g[f"p{degree}_centers"],
                  float(g[f"p{degree}_radius"]), 3, 2, world)
        ctx = DistContext(device="cpu")
        rl, op, x, hx = s.operands(ctx, "cpu")
        s.fill(x, 10 * degree)
        emulated_apply(op, cosine(degree), "h", x, hx)
        parts = ctx.gather((x.to_dense_owned(), hx.to_dense_owned(), len(rl.ghost_groups)))
        if rank == 0:
            xs = np.sum([p[0] for p in parts], axis=0)
            hs = np.sum([p[1] for p in parts], axis=0)
            ghosts = sum(p[2] for p in parts)
            from oracle import numpy_oracle as O

            q.put((bool(np.array_equal(xs, g[f"p{degree}_r2_x"])),
                   O.per_vector_rel_err(hs, g[f"p{degree}_r2_hx"]), ghosts))
        total = ctx.allreduce_sum(float(rank + 1))
        assert total == 3.0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("degree", [1, 2])
def test_two_rank_gloo_apply_matches_reference(degree):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, degree, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    x_equal, err, ghosts = q.get(timeout=10)
    assert x_equal
    assert ghosts > 0  # the exchange really moved data
    assert err <= 1e-12, err

"""Rank contexts: one GPU per rank, messages for setup, buffers for halos.

The reference runs "ranks" as threads exchanging Python objects through
mailboxes (`bcsrmv/comm.py:76-263`).  Here a rank context offers the same
object messaging used by the setup protocols (ghost requests, ordered
allreduce) plus one bulk primitive for device buffers, `exchange()`,
which the ghost update / compress of BlockCsrMatrix use:

* `run_ranks(n, program)` - in-process thread ranks (tests, emulation of a
  multi-GPU run on one device; buffers move as device copies);
* `DistContext` - one process per GPU under torch.distributed: buffers
  move with NCCL point-to-point (NVLink/NVSwitch on a B200 box, grouped
  into one `batch_isend_irecv`), host objects over a gloo side group.
"""

from __future__ import annotations

import json
import pickle
import threading
import time
import zlib
from collections import deque

import numpy as np

from .errors import DeadlockError, DomainError, RankFailure, UsageError

_POLL = 0.02


class _Handle:
    def __init__(self, fn):
        self._fn = fn
        self._done = False

    def wait(self):
        if self._done:
            raise UsageError("handle already waited on")
        self._done = True
        return self._fn()


class RankContext:
    """Common part: ids, ordered collectives built on isend/irecv."""

    rank: int
    n_ranks: int

    def __init__(self):
        self._coll_seq = 0
        self._matrix_seq = 0
        self._xchg_seq = 0

    def next_matrix_id(self) -> int:
        self._matrix_seq += 1
        return self._matrix_seq

    def _next(self) -> int:
        self._coll_seq += 1
        return self._coll_seq

    def allreduce_sum(self, value):
        """Sum with a fixed rank-ascending order (bit-identical on all ranks)."""
        seq = self._next()
        if self.n_ranks == 1:
            return value
        if self.rank == 0:
            acc = value
            for src in range(1, self.n_ranks):
                acc = acc + self.irecv(src, ("_coll", seq)).wait()
            sends = [self.isend(dst, ("_coll_b", seq), acc) for dst in range(1, self.n_ranks)]
            for h in sends:  # complete before returning: a rank may tear down next
                h.wait()
            return acc
        self.isend(0, ("_coll", seq), value)
        return self.irecv(0, ("_coll_b", seq)).wait()

    def barrier(self):
        self.allreduce_sum(0)

    def gather(self, value, root: int = 0):
        seq = self._next()
        if self.rank == root:
            out = [None] * self.n_ranks
            out[root] = value
            for src in range(self.n_ranks):
                if src != root:
                    out[src] = self.irecv(src, ("_gath", seq)).wait()
            return out
        self.isend(root, ("_gath", seq), value).wait()
        return None

    def stream_sync(self):
        pass


# -- in-process thread ranks ------------------------------------------------


class _Runtime:
    def __init__(self, n_ranks: int, timeout: float, trace: bool):
        if n_ranks < 1:
            raise DomainError("need at least one rank")
        self.n_ranks = n_ranks
        self.timeout = timeout
        self.cond = threading.Condition()
        self.queues: list[dict] = [dict() for _ in range(n_ranks)]
        self.blocked = 0
        self.live = n_ranks
        self.activity = 0
        self.trace = [] if trace else None

    def put(self, src, dst, tag, payload):
        if dst < 0 or dst >= self.n_ranks:
            raise DomainError(f"peer {dst} outside [0, {self.n_ranks})")
        with self.cond:
            self.queues[dst].setdefault((src, tag), deque()).append(payload)
            self.activity += 1
            if self.trace is not None:
                self.trace.append({"step": len(self.trace) + 1, "sender": src, "receiver": dst,
                                   "tag": repr(tag), "bytes": _nbytes(payload)})
            self.cond.notify_all()

    def take(self, me, src, tag):
        key = (src, tag)
        idle = 0.0
        with self.cond:
            while True:
                q = self.queues[me].get(key)
                if q:
                    v = q.popleft()
                    if not q:
                        del self.queues[me][key]
                    self.activity += 1
                    return v
                seen = self.activity
                self.blocked += 1
                self.cond.wait(_POLL)
                self.blocked -= 1
                if self.activity != seen:
                    idle = 0.0
                    continue
                idle += _POLL
                if idle >= self.timeout and self.blocked + 1 >= self.live:
                    raise DeadlockError(
                        f"rank {me} blocked on recv(src={src}, tag={tag!r}) with all live "
                        f"ranks idle for {idle:.1f}s")

    def done(self):
        with self.cond:
            self.live -= 1
            self.cond.notify_all()


def _nbytes(payload) -> int:
    if isinstance(payload, np.ndarray):
        return payload.nbytes
    if isinstance(payload, (tuple, list)):
        return sum(_nbytes(p) for p in payload)
    nb = getattr(payload, "nbytes", None)
    return int(nb) if nb is not None else 0


class ThreadRankContext(RankContext):
    def __init__(self, rt: _Runtime, rank: int, device=None):
        super().__init__()
        self._rt = rt
        self.rank = rank
        self.n_ranks = rt.n_ranks
        self.device = device

    def isend(self, peer, tag, payload):
        self._rt.put(self.rank, peer, tag, payload)
        return _Handle(lambda: None)

    def irecv(self, peer, tag):
        if peer < 0 or peer >= self.n_ranks:
            raise DomainError(f"peer {peer} outside [0, {self.n_ranks})")
        return _Handle(lambda: self._rt.take(self.rank, peer, tag))

    def exchange_start(self, sends, recvs, key=None):
        """Post all buffer sends; the receives complete in exchange_finish."""
        self._xchg_seq += 1
        tag = ("_xchg", self._xchg_seq)
        for peer, buf in sends:
            self.isend(peer, tag, buf.clone())
        return (tag, recvs)

    def exchange_finish(self, handle):
        """Fill every receive buffer (in place); ProtocolError on a size mismatch."""
        tag, recvs = handle
        for peer, buf in recvs:
            got = self.irecv(peer, tag).wait()
            if got.numel() != buf.numel():
                from .errors import ProtocolError

                raise ProtocolError(
                    f"rank {self.rank}: buffer from {peer} has {got.numel()} values, "
                    f"expected {buf.numel()}")
            buf.copy_(got)

    def exchange(self, sends, recvs, key=None):
        self.exchange_finish(self.exchange_start(sends, recvs, key))


def run_ranks(n_ranks, program, *shared, deadlock_timeout=30.0, trace_path=None, device=None):
    """Run program(ctx, *shared) on n thread ranks; list of results by rank."""
    rt = _Runtime(n_ranks, deadlock_timeout, trace_path is not None)
    results = [None] * n_ranks
    failures = {}
    if n_ranks == 1:
        results[0] = program(ThreadRankContext(rt, 0, device), *shared)
    else:
        def work(r):
            try:
                _bind_device(device)
                results[r] = program(ThreadRankContext(rt, r, device), *shared)
            except BaseException as exc:  # re-raised on the caller
                failures[r] = exc
            finally:
                rt.done()

        threads = [threading.Thread(target=work, args=(r,), name=f"rank-{r}")
                   for r in range(n_ranks)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if failures:
            primary = {r: e for r, e in failures.items() if not isinstance(e, DeadlockError)}
            raise RankFailure(primary or failures)
    if trace_path is not None:
        with open(trace_path, "w") as fh:
            for rec in rt.trace:
                fh.write(json.dumps(rec) + "\n")
    return results


def _bind_device(device):
    if device is None:
        return
    import torch

    d = torch.device(device)
    if d.type == "cuda":
        torch.cuda.set_device(d)


def serial_context(device=None) -> ThreadRankContext:
    return ThreadRankContext(_Runtime(1, 30.0, False), 0, device)


# -- torch.distributed ranks ---------------------------------------------------


def _tag_int(tag) -> int:
    return zlib.crc32(repr(tag).encode()) & 0x3FFFFFFF


class DistContext(RankContext):
    """Rank context over an initialised torch.distributed process group.

    Device buffers use the default group (NCCL on GPUs, gloo on CPU tests);
    pickled host objects use a gloo side group with tag matching.
    """

    def __init__(self, device=None):
        super().__init__()
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            raise UsageError("torch.distributed is not initialised")
        self._dist = dist
        self.rank = dist.get_rank()
        self.n_ranks = dist.get_world_size()
        self.backend = dist.get_backend()
        self._obj_group = dist.new_group(backend="gloo") if self.backend != "gloo" else None
        self.device = device
        self._pending = []
        self._verified = set()
        self._torch = torch
        # the first NCCL call of a group must involve every rank; point-to-point
        # halo exchanges do not, so initialise the communicator collectively here
        if self.backend == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()

    def isend(self, peer, tag, payload):
        torch = self._torch
        raw = np.frombuffer(pickle.dumps(payload, protocol=pickle.HIGHEST_PROTOCOL),
                            dtype=np.uint8).copy()
        t = _tag_int(tag)
        size = torch.tensor([raw.size], dtype=torch.int64)
        data = torch.from_numpy(raw)
        w1 = self._dist.isend(size, peer, group=self._obj_group, tag=t)
        w2 = self._dist.isend(data, peer, group=self._obj_group, tag=t + 1)
        self._pending.append((w1, w2, size, data))
        return _Handle(lambda: (w1.wait(), w2.wait(), None)[-1])

    def irecv(self, peer, tag):
        if peer < 0 or peer >= self.n_ranks:
            raise DomainError(f"peer {peer} outside [0, {self.n_ranks})")
        torch = self._torch
        t = _tag_int(tag)

        def wait():
            size = torch.zeros(1, dtype=torch.int64)
            self._dist.recv(size, peer, group=self._obj_group, tag=t)
            data = torch.empty(int(size.item()), dtype=torch.uint8)
            self._dist.recv(data, peer, group=self._obj_group, tag=t + 1)
            self._reap()
            return pickle.loads(data.numpy().tobytes())

        return _Handle(wait)

    def _reap(self):
        keep = []
        for item in self._pending:
            if not (item[0].is_completed() and item[1].is_completed()):
                keep.append(item)
        self._pending = keep

    def _verify_sizes(self, sends, recvs, key):
        """Once per exchange plan (key: matrix id and direction, the same on every
        rank): all ranks gather every rank's per-peer send / receive sizes and
        check them pairwise -- ProtocolError instead of an NCCL hang or silent
        corruption."""
        if key is None or key in self._verified:
            return
        mine = ({int(p): int(b.numel()) for p, b in sends},
                {int(p): int(b.numel()) for p, b in recvs})
        tables = [None] * self.n_ranks
        self._dist.all_gather_object(tables, mine, group=self._obj_group)
        for p, (their_send, their_recv) in enumerate(tables):
            if p == self.rank:
                continue
            if mine[0].get(p, 0) != their_recv.get(self.rank, 0) or \
                    mine[1].get(p, 0) != their_send.get(self.rank, 0):
                from .errors import ProtocolError

                raise ProtocolError(
                    f"rank {self.rank}: exchange {key} with rank {p}: I send "
                    f"{mine[0].get(p, 0)} / receive {mine[1].get(p, 0)} values, the peer "
                    f"receives {their_recv.get(self.rank, 0)} / sends "
                    f"{their_send.get(self.rank, 0)}")
        self._verified.add(key)

    def exchange_start(self, sends, recvs, key=None):
        """Post the NCCL (gloo on CPU) point-to-point sends and receives; the
        returned works are waited on in exchange_finish, so kernels launched in
        between overlap the transfer."""
        self._verify_sizes(sends, recvs, key)
        ops = [self._dist.P2POp(self._dist.isend, buf, peer) for peer, buf in sends]
        ops += [self._dist.P2POp(self._dist.irecv, buf, peer) for peer, buf in recvs]
        if not ops:
            return []
        return self._dist.batch_isend_irecv(ops)

    def exchange_finish(self, works):
        for w in works:
            w.wait()

    def exchange(self, sends, recvs, key=None):
        self.exchange_finish(self.exchange_start(sends, recvs, key))

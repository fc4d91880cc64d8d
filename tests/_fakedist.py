"""In-process stand-in for the torch.distributed subset SlabWorld uses (TEST ONLY).

Each rank is a Python thread; point-to-point messages travel through FIFO
mailboxes keyed by (src, dst), all_reduce is a generation-counted barrier.
Lets several slab ranks share ONE GPU in one process so the migration kernels
(b2m_move_migrate / b2m_outbox / b2m_inbox_append) are exercised end to end
without NCCL -- the exchange is host-mediated, no kernel waits on another.
"""
from __future__ import annotations

import collections
import threading

import torch


class ReduceOp:
    SUM = "sum"
    MAX = "max"


P2POp = collections.namedtuple("P2POp", ["op", "tensor", "peer"])


class _World:
    def __init__(self, n):
        self.n = n
        self.cv = threading.Condition()
        self.box = collections.defaultdict(collections.deque)
        self.gen = 0
        self.acc = None
        self.arrived = 0
        self.result = None


def _sync_cuda(t):
    if t.is_cuda:
        torch.cuda.synchronize(t.device)


class _Req:
    def __init__(self, fn):
        self.fn = fn

    def wait(self):
        self.fn()


class FakeDist:
    ReduceOp = ReduceOp
    P2POp = P2POp

    def __init__(self, world: _World, rank: int):
        self.w = world
        self.rank = rank

    @staticmethod
    def make(n):
        w = _World(n)
        return [FakeDist(w, r) for r in range(n)]

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.w.n

    # markers used as P2POp.op
    def isend(self, *a, **k):  # pragma: no cover - marker only
        raise RuntimeError("use batch_isend_irecv")

    def irecv(self, *a, **k):  # pragma: no cover - marker only
        raise RuntimeError("use batch_isend_irecv")

    def batch_isend_irecv(self, ops):
        reqs = []
        for op in ops:
            if op.op == self.isend:
                _sync_cuda(op.tensor)
                with self.w.cv:
                    self.w.box[(self.rank, op.peer)].append(op.tensor.detach().clone())
                    self.w.cv.notify_all()
                reqs.append(_Req(lambda: None))
        for op in ops:
            if op.op == self.irecv:
                def recv(op=op):
                    key = (op.peer, self.rank)
                    with self.w.cv:
                        while not self.w.box[key]:
                            self.w.cv.wait(timeout=60)
                        t = self.w.box[key].popleft()
                    op.tensor.copy_(t.to(op.tensor.device))
                    _sync_cuda(op.tensor)
                reqs.append(_Req(recv))
        return reqs

    def all_reduce(self, t, op=ReduceOp.SUM):
        w = self.w
        v = t.detach().cpu().clone()
        with w.cv:
            gen = w.gen
            w.acc = v if w.acc is None else (w.acc + v if op == ReduceOp.SUM
                                             else torch.maximum(w.acc, v))
            w.arrived += 1
            if w.arrived == w.n:
                w.result = w.acc
                w.acc = None
                w.arrived = 0
                w.gen += 1
                w.cv.notify_all()
            else:
                while w.gen == gen:
                    w.cv.wait(timeout=60)
            res = w.result
        t.copy_(res.to(t.device))


def run_ranks(fn, n):
    """Run fn(rank, dist) on n threads; return per-rank results or raise the
    first exception."""
    dists = FakeDist.make(n)
    out = [None] * n
    errs = [None] * n

    def body(r):
        try:
            out[r] = fn(r, dists[r])
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    return out, errs

"""Partition layer: y-slab domain decomposition across GPUs (one process per
GPU) with NCCL particle migration -- the B200 equivalent of the reference's
multi-worker ``Simulation`` (runtime.cpp:22-76, :211-289).

* ``decompose`` / ``owner_of`` are the reference's slab rules
  (runtime.cpp:22-44), with the same ConfigError texts.
* ``SlabWorld`` drives one rank: the mover kernel is fused with the owner scan
  (``b2m_move_migrate``), leavers go to the prev/next outboxes, counts then
  payloads are exchanged with ``torch.distributed`` point-to-point ops (NCCL
  over NVLink on GPUs), arrivals fill the holes the leavers left
  (``b2m_inbox_append``), and an all-reduce checks particle-count conservation
  (runtime.cpp:264-269).  A particle that lands farther than one slab away
  raises CflViolation (runtime.cpp:55-59).
* The field is replicated: rank 0's field is broadcast each cycle
  (runtime.cpp:143 keeps a full copy per worker).

The exchange code only needs a *store* with the DeviceStore migration methods
and a torch device, so the same protocol runs over gloo with a host test
double (tests/test_partition.py).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, EngineFault


@dataclass(frozen=True)
class Subdomain:
    """One worker's y-slab [j_lo, j_hi) with periodic neighbours (runtime.hpp:13-20)."""
    worker_id: int
    j_lo: int
    j_hi: int
    prev: int
    next: int


def decompose(grid, workers: int):
    """Equal slabs along y (runtime.cpp:22-37)."""
    if workers < 1:
        raise ConfigError("workers: must be >= 1")
    if grid.ny % workers != 0:
        raise ConfigError(f"workers: {workers} does not divide ny={grid.ny}")
    slab = grid.ny // workers
    if slab < 2:
        raise ConfigError(f"workers: slab would be {slab} cells; each slab needs at least 2")
    return [Subdomain(w, w * slab, (w + 1) * slab, (w + workers - 1) % workers, (w + 1) % workers)
            for w in range(workers)]


def owner_of(y, grid, workers: int):
    """Owner worker of wrapped y coordinate(s) (runtime.cpp:39-44):
    j = int(y/dy) (truncation), clamped to [0, ny-1], then j / slab.
    Vectorised over numpy arrays."""
    y = np.asarray(y, dtype=np.float64)
    j = np.trunc(y / grid.dy)
    j = np.where(np.isnan(j), 0, j)
    j = np.clip(j, 0, grid.ny - 1).astype(np.int64)
    return j // (grid.ny // workers)


class _CudaArray:
    """Zero-copy torch view of a libb2m device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, stream: int = 0):
        # no "stream" entry: the producer (b2m_sync) has already completed
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": None}


class DeviceMigration:
    """Migration methods of a GPU DeviceStore (C ABI b2m_slab_config /
    b2m_move_migrate / b2m_outbox / b2m_inbox_append)."""

    def __init__(self, store, rank: int, world: int):
        from . import _capi
        self._capi = _capi
        self.store = store
        _capi.check(_capi.lib().b2m_slab_config(store.h, rank, world))

    def move_migrate(self, s: int, mp):
        self._capi.check(self._capi.lib().b2m_move_migrate(self.store.h, s, C.byref(mp.to_c())))

    def move_migrate_all(self, mps):
        arr = (self._capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
        self._capi.check(self._capi.lib().b2m_move_migrate_all(self.store.h, arr))

    def outbox(self, s: int, direction: int):
        import torch
        p = C.c_void_p()
        n = C.c_uint64()
        self._capi.check(self._capi.lib().b2m_outbox(self.store.h, s, direction, C.byref(p),
                                                     C.byref(n)))
        if n.value == 0:
            if getattr(self, "_empty", None) is None:
                self._empty = torch.empty((0, 6), dtype=torch.float64, device="cuda")
            return self._empty
        return torch.as_tensor(_CudaArray(p.value, (n.value, 6)), device="cuda")

    def inbox_append(self, s: int, recs):
        n = int(recs.shape[0])
        ptr = recs.data_ptr() if n else 0
        self._capi.check(self._capi.lib().b2m_inbox_append(self.store.h, s, C.c_void_p(ptr), n))

    def sync(self):
        self.store.sync()

    def count(self, s: int) -> int:
        return self.store.count(s)

    # moments of this rank's particles (b2m_deposit), as a device tensor
    def moments_zero(self, with_pressure: bool = False):
        self.store.moments_zero(with_pressure)

    def deposit(self, s: int, q_per_particle: float):
        self.store.deposit(s, q_per_particle)

    def moments_tensor(self):
        import torch
        ptr, n = self.store.moments_device()
        return torch.as_tensor(_CudaArray(ptr, (n,)), device="cuda")


class SlabWorld:
    """One rank of the slab-partitioned mover.

    ``store`` provides move_migrate / outbox / inbox_append / sync / count
    (DeviceMigration on GPUs); ``dist`` is torch.distributed (initialised);
    ``device`` the torch device of the exchanged tensors."""

    def __init__(self, grid, store, n_species: int, dist, device):
        self.grid = grid
        self.store = store
        self.ns = n_species
        self.dist = dist
        self.device = device
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.subs = decompose(grid, self.world)
        me = self.subs[self.rank]
        self.prev, self.next = me.prev, me.next
        self.total = None
        self.last_exchange = {}
        # gloo has no CUDA point-to-point: stage device tensors through host
        backend = getattr(dist, "get_backend", lambda: "")()
        self.stage_host = (str(backend) == "gloo" and getattr(device, "type", "") == "cuda")

    def _reduce_count(self, count: int, faulted: int):
        """Global (count, faulted ranks): one all-reduce of two int64 through
        reused pinned-host / device buffers (no pageable copy per cycle)."""
        import torch
        if getattr(self, "_cnt_dev", None) is None:
            pin = getattr(self.device, "type", "") == "cuda"
            self._cnt_host = torch.empty(2, dtype=torch.int64, pin_memory=pin)
            self._cnt_dev = torch.empty(2, dtype=torch.int64, device=self.device)
        self._cnt_host[0] = count
        self._cnt_host[1] = faulted
        self._cnt_dev.copy_(self._cnt_host, non_blocking=True)
        self._all_reduce(self._cnt_dev)
        self._cnt_host.copy_(self._cnt_dev)  # synchronises
        return int(self._cnt_host[0]), int(self._cnt_host[1])

    def _count_all(self) -> int:
        return sum(self.store.count(s) for s in range(self.ns))

    def set_total(self) -> int:
        """Global particle count (the conservation reference, runtime.cpp:150)."""
        import torch
        t = torch.tensor([self._count_all()], dtype=torch.int64, device=self.device)
        self._all_reduce(t)
        self.total = int(t.item())
        return self.total

    def _all_reduce(self, t, op=None):
        if self.stage_host:
            h = t.cpu()
            self.dist.all_reduce(h) if op is None else self.dist.all_reduce(h, op=op)
            t.copy_(h.to(t.device))
        else:
            self.dist.all_reduce(t) if op is None else self.dist.all_reduce(t, op=op)

    def _exchange(self, outs):
        """Migration of all species in one round trip: ``outs[s] = (to_prev,
        to_next)`` (n, 6) float64 tensors; returns, per species, the (m, 6)
        records that arrive from prev then next."""
        if self.stage_host:
            ins = self._exchange_on([(a.cpu(), b.cpu()) for a, b in outs], "cpu")
            return [t.to(self.device) for t in ins]
        return self._exchange_on(outs, self.device)

    def _exchange_on(self, outs, dev):
        """Counts first (one int64 row per direction and species), then one
        payload per neighbour with every species concatenated: two grouped
        ncclSend/ncclRecv rounds per cycle however many species.  With two
        ranks prev == next and both directions travel in one message."""
        import torch
        dist = self.dist
        ns = len(outs)
        empty = torch.empty((0, 6), dtype=torch.float64, device=dev)
        if self.world == 1:
            return [empty for _ in range(ns)]  # periodic self-neighbour: no leavers
        cnt_out = torch.tensor([[int(a.shape[0]) for a, _ in outs],
                                [int(b.shape[0]) for _, b in outs]], dtype=torch.int64, device=dev)
        pay_prev = [a for a, _ in outs if a.shape[0]]
        pay_next = [b for _, b in outs if b.shape[0]]
        pay_prev = torch.cat(pay_prev, dim=0) if pay_prev else empty
        pay_next = torch.cat(pay_next, dim=0) if pay_next else empty

        def wait_all(ops):
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()

        def split(buf, counts):
            parts, o = [], 0
            for c in counts:
                parts.append(buf[o:o + c])
                o += c
            return parts

        if self.world == 2:
            other = self.prev
            cnt_in = torch.zeros((2, ns), dtype=torch.int64, device=dev)
            wait_all([dist.P2POp(dist.isend, cnt_out, other),
                      dist.P2POp(dist.irecv, cnt_in, other)])
            c_in = cnt_in.cpu().tolist()       # [the other's to-prev, to-next] = both to me
            out = torch.cat([pay_prev, pay_next], dim=0).contiguous()
            n_in = sum(c_in[0]) + sum(c_in[1])
            buf = torch.empty((n_in, 6), dtype=torch.float64, device=dev)
            ops = []
            if out.shape[0]:
                ops.append(dist.P2POp(dist.isend, out, other))
            if n_in:
                ops.append(dist.P2POp(dist.irecv, buf, other))
            wait_all(ops)
            a = split(buf[:sum(c_in[0])], c_in[0])
            b = split(buf[sum(c_in[0]):], c_in[1])
            return [torch.cat([x, y], dim=0) if y.shape[0] else x for x, y in zip(a, b)]

        c_from_prev = torch.zeros(ns, dtype=torch.int64, device=dev)
        c_from_next = torch.zeros(ns, dtype=torch.int64, device=dev)
        wait_all([dist.P2POp(dist.isend, cnt_out[0].clone(), self.prev),
                  dist.P2POp(dist.isend, cnt_out[1].clone(), self.next),
                  dist.P2POp(dist.irecv, c_from_prev, self.prev),
                  dist.P2POp(dist.irecv, c_from_next, self.next)])
        cp, cn = c_from_prev.cpu().tolist(), c_from_next.cpu().tolist()
        from_prev = torch.empty((sum(cp), 6), dtype=torch.float64, device=dev)
        from_next = torch.empty((sum(cn), 6), dtype=torch.float64, device=dev)
        ops = []
        if pay_prev.shape[0]:
            ops.append(dist.P2POp(dist.isend, pay_prev.contiguous(), self.prev))
        if pay_next.shape[0]:
            ops.append(dist.P2POp(dist.isend, pay_next.contiguous(), self.next))
        if from_prev.shape[0]:
            ops.append(dist.P2POp(dist.irecv, from_prev, self.prev))
        if from_next.shape[0]:
            ops.append(dist.P2POp(dist.irecv, from_next, self.next))
        wait_all(ops)
        a, b = split(from_prev, cp), split(from_next, cn)
        return [torch.cat([x, y], dim=0) if y.shape[0] else x for x, y in zip(a, b)]

    def deposit_moments(self, q_per_particle, with_pressure: bool = False):
        """Moments of every rank's particles summed over the ranks into every
        rank's mesh: the reference's per-worker private meshes added up by
        worker 0 (runtime.cpp:251-262), as one all-reduce of the device mesh."""
        st = self.store
        st.moments_zero(with_pressure)
        for s in range(self.ns):
            st.deposit(s, q_per_particle[s])
        st.sync()   # DomainError, as the reference raises it
        mesh = st.moments_tensor()
        self._all_reduce(mesh)
        return mesh

    def step(self, mps, check_counts: bool = True):
        """One mover cycle over all species with migration
        (runtime.cpp:227-244 mover + exchange, :264-269 count check).

        A fault on any rank (NumericalFault, CflViolation, ...) must not
        deadlock its peers inside the exchange (the reference drops the
        faulting worker from the barrier, runtime.cpp:283-288): the faulting
        rank keeps running the protocol with empty outboxes, and the fault
        flag rides on the count all-reduce, after which every rank raises --
        the faulting one its typed error, the others EngineFault."""
        import torch
        st = self.store
        err = None
        try:
            if hasattr(st, "move_migrate_all"):
                st.move_migrate_all(mps)   # one mover launch for every species
            else:
                for s in range(self.ns):
                    st.move_migrate(s, mps[s])
            st.sync()   # NumericalFault / CflViolation, as the reference raises them
        except Exception as e:  # noqa: BLE001 - re-raised after the collective below
            err = e
        empty = torch.empty((0, 6), dtype=torch.float64, device=self.device)
        outs = []
        for s in range(self.ns):
            if err is None:
                try:
                    outs.append((st.outbox(s, 0), st.outbox(s, 1)))
                    continue
                except Exception as e:  # noqa: BLE001
                    err = e
            outs.append((empty, empty))
        if err is not None:   # a faulted rank still takes part, with empty outboxes
            outs = [(empty, empty)] * self.ns
        ins = self._exchange(outs)
        moved = sum(int(a.shape[0] + b.shape[0]) for a, b in outs)
        if err is None:
            for s in range(self.ns):
                try:
                    st.inbox_append(s, ins[s].contiguous())
                except Exception as e:  # noqa: BLE001
                    err = e
                    break
        self.last_exchange = {"sent": moved}
        n, n_faulted = self._reduce_count(self._count_all() if err is None else 0,
                                          1 if err is not None else 0)
        if err is not None:
            raise err
        if n_faulted:
            raise EngineFault(f"simulation aborted: {n_faulted} peer rank(s) faulted in this cycle")
        if check_counts and self.total is not None and n != self.total:
            raise EngineFault(f"particle count drifted: {n} vs {self.total}")
        return moved


class NativeSlabWorld:
    """One rank of the slab-partitioned mover with the whole per-cycle
    protocol in the native library (b2m_world_step: mover + owner scan +
    compaction, counts exchanged with prev / next, the (count, failed)
    all-reduce, then records exchanged and merged -- one host
    synchronisation per step, no Python on the data path).

    ``dist`` (torch.distributed, initialised) only carries the NCCL unique
    id from rank 0 to the others; ``store`` is this rank's DeviceStore."""

    def __init__(self, grid, store, rank: int, world: int, dist=None, comm: bool | None = None):
        from . import _capi
        self._capi = _capi
        self.grid, self.store, self.rank, self.world = grid, store, rank, world
        self.ns = store.n_species
        self.last_exchange = {}
        self.total = None
        uid = (C.c_ubyte * 128)()
        # comm: create an NCCL communicator (default: world > 1; a one-rank
        # communicator runs the same collectives with no peers)
        comm = world > 1 if comm is None else comm
        if comm and dist is None and world > 1:
            raise ConfigError("NativeSlabWorld: world > 1 needs torch.distributed (dist) to "
                              "share the NCCL unique id")
        if comm:
            # every rank probes NCCL (resolved at run time) and the ranks agree
            # before any of them enters ncclCommInitRank: a rank without NCCL
            # makes ALL of them raise ConfigError instead of leaving the others
            # waiting in the communicator setup
            st = (_capi.lib().b2m_world_id(uid) if rank == 0
                  else _capi.lib().b2m_world_nccl_available())
            why = "" if st == 0 else (_capi.last_error() or "NCCL unavailable")
            if dist is not None and world > 1:
                votes = [None] * world
                dist.all_gather_object(votes, why)
                bad = [(r, w) for r, w in enumerate(votes) if w]
                if bad:
                    raise ConfigError(f"native world unavailable (rank {bad[0][0]}: {bad[0][1]})")
            elif why:
                raise ConfigError(f"native world unavailable: {why}")
            if dist is not None:
                obj = [bytes(uid)]
                dist.broadcast_object_list(obj, src=0)
                uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
            _capi.check(_capi.lib().b2m_world_init(store.h, uid, rank, world))
        else:
            _capi.check(_capi.lib().b2m_world_init(store.h, None, rank, world))

    def deposit_moments(self, q_per_particle, with_pressure: bool = False):
        """Moments of every rank's particles summed over the ranks into every
        rank's device mesh (runtime.cpp:251-262); returns the mesh as a tensor."""
        st = self.store
        st.moments_zero(with_pressure)
        for s in range(self.ns):
            st.deposit(s, q_per_particle[s])
        self._capi.check(self._capi.lib().b2m_world_reduce_moments(st.h))
        st.sync()   # DomainError, as the reference raises it
        import torch
        ptr, n = st.moments_device()
        return torch.as_tensor(_CudaArray(ptr, (n,)), device="cuda")

    def broadcast_field(self, root: int = 0) -> None:
        """Replicate the root rank's device field on every rank (NCCL)."""
        self._capi.check(self._capi.lib().b2m_world_broadcast_field(self.store.h, root))

    def set_total(self) -> int:
        n = C.c_uint64()
        self._capi.check(self._capi.lib().b2m_world_set_total(self.store.h, C.byref(n)))
        self.total = int(n.value)
        return self.total

    def step(self, mps) -> int:
        arr = (self._capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
        sent, total = C.c_uint64(), C.c_uint64()
        self._capi.check(self._capi.lib().b2m_world_step(self.store.h, arr, C.byref(sent),
                                                          C.byref(total)))
        self.last_exchange = {"sent": int(sent.value), "global_count": int(total.value)}
        return int(sent.value)


def loopback_world(stores, grid):
    """b2m_world_init (no communicator) on each of ``stores`` as ranks
    0..W-1 of one process: for b2m_world_loopback_step."""
    from . import _capi
    w = len(stores)
    for r, st in enumerate(stores):
        _capi.check(_capi.lib().b2m_world_init(st.h, None, r, w))
        _capi.check(_capi.lib().b2m_world_set_total(st.h, None))


def loopback_step(stores, mps) -> int:
    """One protocol step over in-process ranks (device copies stand in for
    NCCL; the same native phases as b2m_world_step)."""
    from . import _capi
    arr = (_capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
    hs = (C.c_void_p * len(stores))(*[st.h for st in stores])
    sent = C.c_uint64()
    _capi.check(_capi.lib().b2m_world_loopback_step(hs, len(stores), arr, C.byref(sent)))
    return int(sent.value)

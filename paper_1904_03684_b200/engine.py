"""Engine-level boundary: the B200 drop-in for ``pic::Engine``.

``DeviceStore`` owns one ``b2m_ctx`` (one GPU's resident particle SoA, field
buffers and stream) -- the native replacement of the reference's
DeviceArena + CommandQueue (device_arena.cpp:17-111, command_queue.cpp:9-95).

``B200Engine`` implements the reference Engine contract (engines.hpp:20-48):
``prime`` / ``stage_next`` / ``run_mover`` with the same blocking semantics,
host batches updated on return, faults surfaced as ``EngineFault`` that poison
the engine (test_offload.cpp:464-481).
"""
from __future__ import annotations

import ctypes as C

from . import _capi
from .errors import EngineFault, MinipicError, NumericalFault
from .mover import MODES, FieldMesh, Grid, MoverParams


class DeviceStore:
    """One context: species capacities fixed at creation (AllocError there,
    never mid-run, like DeviceArena::configure)."""

    def __init__(self, grid: Grid, capacities, mode="fast", device: int = 0):
        self.grid = grid
        self.n_species = len(capacities)
        self.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        caps = (C.c_uint64 * max(1, self.n_species))(*[int(c) for c in capacities])
        h = C.c_void_p()
        self._g = grid.to_c()
        _capi.check(_capi.lib().b2m_ctx_create(device, C.byref(self._g), self.n_species, caps,
                                               self.mode, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().b2m_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library may be gone already
            pass

    # -- plumbing -----------------------------------------------------------
    def set_stream(self, stream_handle: int | None):
        _capi.check(_capi.lib().b2m_ctx_set_stream(self.h, C.c_void_p(stream_handle or 0)))

    def set_mode(self, mode):
        self.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        _capi.check(_capi.lib().b2m_ctx_set_mode(self.h, self.mode))

    def upload_field(self, field: FieldMesh):
        _capi.check(_capi.lib().b2m_field_upload(self.h, _capi.dptr(field.E), _capi.dptr(field.B),
                                                 field.node_count()))

    def field_stub(self, passes: int):
        """field_phase_stub on the device field (kernels.cpp:185-215)."""
        _capi.check(_capi.lib().b2m_field_phase_stub(self.h, int(passes)))

    def download_field(self, field: FieldMesh):
        _capi.check(_capi.lib().b2m_field_download(self.h, _capi.dptr(field.E),
                                                   _capi.dptr(field.B)))

    def upload_field_device(self, dE: int, dB: int):
        _capi.check(_capi.lib().b2m_field_upload_device(self.h, C.c_void_p(dE), C.c_void_p(dB),
                                                        self.grid.nodes()))

    def field_device_ptrs(self):
        """(dE, dB) device pointers of this context's field buffers."""
        e, b = C.c_void_p(), C.c_void_p()
        _capi.check(_capi.lib().b2m_field_device_ptrs(self.h, C.byref(e), C.byref(b)))
        return int(e.value), int(b.value)

    def kernel_timing_begin(self, n: int):
        """Log the mover-launch time of the next n move_all calls (no syncs)."""
        _capi.check(_capi.lib().b2m_kernel_timing_begin(self.h, n))

    def kernel_timing_read(self, max_n: int = 1 << 16):
        buf = (C.c_float * max_n)()
        n = C.c_int()
        _capi.check(_capi.lib().b2m_kernel_timing_read(self.h, buf, max_n, C.byref(n)))
        return [float(buf[i]) for i in range(n.value)]

    def field_changed(self):
        """The device field was rewritten in place (a device-side field phase):
        the gather tables rebuild on the next move (no copy)."""
        self.upload_field_device(*self.field_device_ptrs())

    def upload(self, s: int, p6, n: int | None = None):
        n = len(p6[0]) if n is None else n
        _capi.check(_capi.lib().b2m_species_upload(self.h, s, _capi.ptr6(p6), n))

    def download(self, s: int, p6) -> int:
        n = C.c_uint64()
        _capi.check(_capi.lib().b2m_species_download(self.h, s, _capi.ptr6(p6), len(p6[0]),
                                                     C.byref(n)))
        return n.value

    def download_range(self, s: int, p6, offset: int, n: int):
        """Particles [offset, offset + n) of species s into host arrays."""
        _capi.check(_capi.lib().b2m_species_download_range(self.h, s, _capi.ptr6(p6), offset, n))

    def count(self, s: int) -> int:
        n = C.c_uint64()
        _capi.check(_capi.lib().b2m_species_count(self.h, s, C.byref(n)))
        return n.value

    def device_ptrs(self, s: int):
        out = (C.c_void_p * 6)()
        _capi.check(_capi.lib().b2m_species_device_ptrs(self.h, s, out))
        return [int(p) for p in out]

    def move(self, s: int, mp: MoverParams):
        _capi.check(_capi.lib().b2m_move(self.h, s, C.byref(mp.to_c())))

    def move_all(self, mps):
        arr = (_capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
        _capi.check(_capi.lib().b2m_move_all(self.h, arr))

    def move_deposit_all(self, mps, q_per_particle):
        """One mover cycle of every species and the deposition of rho, J (and
        the pressure tensor when the mesh has it) of the new state into the
        moment mesh (b2m_moments_zero first).  FAST without pressure: one
        fused launch (b2m_move_deposit_all)."""
        arr = (_capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
        q = (C.c_double * len(mps))(*[float(x) for x in q_per_particle])
        _capi.check(_capi.lib().b2m_move_deposit_all(self.h, arr, q))

    def run_mover_host(self, batches, mps, chunk: int = 1 << 21):
        """Chunked H2D -> kernel -> D2H over three streams (b2m_run_mover_host)."""
        ns = len(batches)
        ptrs = (_capi._dp * (6 * ns))(*[_capi.dptr(a) for b in batches for a in b.arrays])
        counts = (C.c_uint64 * ns)(*[b.count() for b in batches])
        arr = (_capi.b2m_mover_params * ns)(*[m.to_c() for m in mps])
        st = _capi.lib().b2m_run_mover_host(self.h, ns, ptrs, counts, arr, chunk)
        if st == 4:
            raise NumericalFault(_capi.last_error())
        _capi.check(st)

    def sort(self, s: int):
        _capi.check(_capi.lib().b2m_sort_species(self.h, s))

    def sync(self):
        """Wait for the stream; raise NumericalFault / CflViolation recorded by
        the kernels (the context is poisoned afterwards)."""
        bs = C.c_int(-1)
        bi = C.c_int64(-1)
        st = _capi.lib().b2m_sync(self.h, C.byref(bs), C.byref(bi))
        if st == 4:
            raise NumericalFault(_capi.last_error(), index=bi.value, species=bs.value)
        _capi.check(st)

    # -- moments (deposit_moments, kernels.cpp:147-183) -----------------------
    def moments_zero(self, with_pressure: bool = False):
        _capi.check(_capi.lib().b2m_moments_zero(self.h, int(with_pressure)))

    def deposit(self, s: int, q_per_particle: float):
        _capi.check(_capi.lib().b2m_deposit(self.h, s, float(q_per_particle)))

    def moments_device(self):
        """(device pointer, n_doubles) of the contiguous device moment mesh."""
        p = _capi._dp()
        n = C.c_uint64()
        _capi.check(_capi.lib().b2m_moments_device_ptr(self.h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, n.value

    def moments_download(self, mesh) -> None:
        """Copy the device moment mesh into ``mesh`` (a MomentMesh) and sync."""
        ptrs = (_capi._dp * len(mesh.arrays))(*[_capi.dptr(a) for a in mesh.arrays])
        _capi.check(_capi.lib().b2m_moments_download(self.h, ptrs, len(mesh.arrays)))

    def record(self, slot: int):
        _capi.check(_capi.lib().b2m_event_record(self.h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _capi.check(_capi.lib().b2m_event_elapsed_ms(self.h, a, b, C.byref(ms)))
        return ms.value


class B200Engine:
    """pic::Engine on one B200 (engines.hpp:20-48).

    schedule "sync": field up, then per species up / kernel / down, like the
    reference SyncEngine (engines.cpp:138-150); "prefetch": the field and
    species 0 are staged in ``stage_next`` (engines.cpp:169-173) so they
    overlap the host's phases; "pipeline" (default): the field is staged in
    ``stage_next`` and every species flows through chunked H2D / kernel / D2H
    on three streams (b2m_run_mover_host), so both PCIe directions and the
    kernel overlap -- the prefetch idea of PAPER.md:96-98 at chunk grain.  Results are bit-identical to the reference in
    mode "strict" and within the 1e-12 contract in mode "fast"."""

    def __init__(self, grid: Grid, mode="fast", schedule="pipeline", device: int = 0,
                 chunk: int = 1 << 21):
        self.grid = grid
        self.mode = mode
        self.schedule = schedule
        self.device = device
        self.chunk = chunk
        self.store: DeviceStore | None = None
        self._staged = False
        self._poisoned = None

    def kind(self) -> str:
        return "b200-" + self.schedule

    def _check_poison(self):
        if self._poisoned is not None:
            raise EngineFault("engine state is invalid after an earlier fault: " + self._poisoned)

    def prime(self, field: FieldMesh, batches):
        """Lay out device memory for every batch's capacity (untimed)."""
        self.store = DeviceStore(self.grid, [b.capacity() for b in batches], self.mode,
                                 self.device)
        if self.schedule in ("prefetch", "pipeline"):
            self.stage_next(field, batches)
            self._sync()

    def stage_next(self, field: FieldMesh, batches):
        if self.schedule not in ("prefetch", "pipeline"):
            return
        self._check_poison()
        self.store.upload_field(field)
        if batches and self.schedule == "prefetch":
            self.store.upload(0, batches[0].span())
        self._staged = True

    def close(self):
        if self.store is not None:
            self.store.close()
            self.store = None

    def _sync(self):
        try:
            self.store.sync()
        except MinipicError as e:
            self._poisoned = str(e)
            raise EngineFault(str(e)) from e

    def run_mover(self, field: FieldMesh, batches, mps):
        self._check_poison()
        if self.store is None:
            self.prime(field, batches)
        st = self.store
        if self.schedule == "pipeline":
            try:
                if not self._staged:
                    st.upload_field(field)
                self._staged = False
                st.run_mover_host(batches, mps, self.chunk)
            except MinipicError as e:
                self._poisoned = str(e)
                raise EngineFault(str(e)) from e
            return
        try:
            if not self._staged:
                st.upload_field(field)
                if batches:
                    st.upload(0, batches[0].span())
            self._staged = False
            for s, b in enumerate(batches):
                if s > 0:
                    st.upload(s, b.span())
                st.move(s, mps[s])
                if self.schedule == "sync":
                    self._sync()
            self._sync()
            for s, b in enumerate(batches):
                st.download(s, b.arrays)
            self._sync()
        except EngineFault:
            raise
        except MinipicError as e:
            self._poisoned = str(e)
            raise EngineFault(str(e)) from e

"""Python mirror of the reference's tile API over the C ABI.

Names, argument meaning and error behaviour follow xbarsim
(``proj/include/xbarsim/tile.hpp:47-131``, ``compound.hpp:73-131``,
``inference.hpp:21-93``) so the parity tests read like the reference's own
tests.  Every method also accepts a batch: ``forward(X)`` with ``X`` of shape
``(B, d_in)`` equals B sequential reference calls.

Host (numpy) inputs go through the synchronous host-buffer entries; the
``*_dev`` methods take CUDA tensors (anything with ``data_ptr()``) and run
asynchronously on the tile's stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _abi
from ._abi import (DeviceParams, InferenceModel, IOParams, Shard, TemporalParams, TileConfig,
                   TransferConfig, UnitCellConfig, UpdateParams)

_lib = _abi.load()

_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)


class Error(RuntimeError):
    """Mirror of xbarsim::Error (proj/include/xbarsim/common.hpp:15-18)."""


def _check(rc: int) -> None:
    if rc != 0:
        raise Error(_lib.xb_last_error().decode())


def lib():
    return _lib


def launch_count() -> int:
    return int(_lib.xb_launch_count())


def launch_floor_us(n: int = 64, reps: int = 5) -> float:
    """Device microseconds per launch of n empty kernels issued back to back
    from C (include/xbtile.h: xb_launch_floor_us)."""
    out = C.c_double()
    _check(_lib.xb_launch_floor_us(int(n), int(reps), C.byref(out)))
    return out.value


def device_check() -> None:
    _check(_lib.xb_device_check())


# ------------------------------------------------------------------ settings
def default_device() -> DeviceParams:
    p = DeviceParams()
    _lib.xb_default_device(C.byref(p))
    return p


def default_io() -> IOParams:
    p = IOParams()
    _lib.xb_default_io(C.byref(p))
    return p


def perfect_io() -> IOParams:
    """proj/src/io.cpp:32-40."""
    p = IOParams()
    _lib.xb_perfect_io(C.byref(p))
    return p


def io_off() -> IOParams:
    """The reference tests' io_off(): full analog path, non-idealities off
    (proj/tests/helpers.hpp:56-68)."""
    io = default_io()
    io.dac_bits, io.adc_bits = 0, 0
    io.input_bound, io.output_bound = 1e9, 1e9
    io.sigma_inp = io.sigma_out = io.sigma_w = 0.0
    io.noise_management = _abi.NM_NONE
    io.is_perfect = 0
    return io


def device_preset(name: str) -> DeviceParams:
    """proj/src/device.cpp:100-132."""
    p = DeviceParams()
    _check(_lib.xb_device_preset(name.encode(), C.byref(p)))
    return p


def TileSettings(device: Optional[DeviceParams] = None, forward_io: Optional[IOParams] = None,
                 backward_io: Optional[IOParams] = None, update: Optional[UpdateParams] = None,
                 temporal: Optional[TemporalParams] = None,
                 mvm_precision: int = _abi.MVM_TF32X3,
                 weight_precision: int = _abi.W_AUTO) -> TileConfig:
    """proj/include/xbarsim/tile.hpp:38-44 with reference defaults."""
    c = TileConfig()
    _lib.xb_default_config(C.byref(c))
    if device is not None:
        c.device = device
    if forward_io is not None:
        c.forward_io = forward_io
    if backward_io is not None:
        c.backward_io = backward_io
    if update is not None:
        c.update = update
    if temporal is not None:
        c.temporal = temporal
    c.mvm_precision = mvm_precision
    c.weight_precision = weight_precision
    return c


def TransferSettings() -> TransferConfig:
    c = TransferConfig()
    _lib.xb_default_transfer_config(C.byref(c))
    return c


def UnitCellSettings(devices=None, gains=None, policy: int = _abi.UC_ALL_TOGETHER,
                     forward_io: Optional[IOParams] = None, backward_io: Optional[IOParams] = None,
                     update: Optional[UpdateParams] = None,
                     temporal: Optional[TemporalParams] = None,
                     mvm_precision: int = _abi.MVM_TF32X3) -> UnitCellConfig:
    """proj/include/xbarsim/compound.hpp:15-28 with reference defaults
    (one default device of gain 1, all_together)."""
    c = UnitCellConfig()
    _lib.xb_default_unitcell_config(C.byref(c))
    if devices is not None:
        devices = list(devices)
        gains = [1.0] * len(devices) if gains is None else list(gains)
        if len(devices) > _abi.MAX_CELL_DEVICES:
            raise Error(f"unit_cell.devices: at most {_abi.MAX_CELL_DEVICES} on the B200 path")
        c.n_devices = len(devices)
        for k, d in enumerate(devices):
            c.devices[k] = d
        if len(gains) != len(devices):
            raise Error("unit_cell.gains: length must match devices")
        for k, g in enumerate(gains):
            c.gains[k] = float(g)
    c.policy = policy
    for name, v in (("forward_io", forward_io), ("backward_io", backward_io),
                    ("update", update), ("temporal", temporal)):
        if v is not None:
            setattr(c, name, v)
    c.mvm_precision = mvm_precision
    return c


def InferenceNoiseModel() -> InferenceModel:
    m = InferenceModel()
    _lib.xb_default_inference_model(C.byref(m))
    return m


# ------------------------------------------------------------------ helpers
def _f32(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if shape is not None and a.shape != shape:
        raise Error(f"shape {a.shape}, expected {shape}")
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_fp)


def _batch(x, n: int, what: str):
    """(n,) or (B, n) -> (B, n) contiguous fp32, squeeze flag."""
    a = np.asarray(x, dtype=np.float32)
    single = a.ndim == 1
    a = np.ascontiguousarray(a.reshape(1, -1) if single else a)
    if a.ndim != 2 or a.shape[1] != n:
        raise Error(f"{what}: length {a.shape[-1]}, expected {n}")
    return a, single


def _out(out, shape) -> np.ndarray:
    if out is None:
        return np.empty(shape, dtype=np.float32)
    if (not isinstance(out, np.ndarray) or out.dtype != np.float32 or
            not out.flags["C_CONTIGUOUS"] or out.size != shape[0] * shape[1]):
        raise Error(f"out: need a C-contiguous float32 array of {shape[0]}x{shape[1]}")
    return out


_LR_CACHE = {}


def _lr_array(lr, B: int):
    if lr is None:
        return None
    # the reference takes double lr (proj/include/xbarsim/tile.hpp:84); no narrowing
    if np.ndim(lr) == 0:  # a scalar: the same B-vector every call (kept, read-only)
        key = (float(lr), B)
        hit = _LR_CACHE.get(key)
        if hit is None:
            if len(_LR_CACHE) > 64:
                _LR_CACHE.clear()
            arr = np.full(B, float(lr), dtype=np.float64)
            arr.setflags(write=False)
            hit = _LR_CACHE[key] = (arr.ctypes.data_as(_dp), arr)
        return hit
    arr = np.ascontiguousarray(np.broadcast_to(np.asarray(lr, dtype=np.float64), (B,)))
    return arr.ctypes.data_as(_dp), arr


def _tptr(t) -> int:
    return C.c_void_p(t.data_ptr())


class Comm:
    """Communicator of a row-sharded tile (include/xbtile.h: xb_comm_*).

    ``Comm.unique_id()`` on rank 0, sent to the other ranks out of band, then
    ``Comm(uid, nranks, rank)`` on every rank (NCCL, current CUDA device);
    ``Comm.local(n)`` is an in-process group of n handles, one per host thread
    driving one shard (loopback, for tests on one device)."""

    def __init__(self, uid: Optional[bytes] = None, nranks: int = 1, rank: int = 0, _h=None):
        if _h is not None:
            self._h = _h
            return
        if uid is None or len(uid) != _abi.COMM_ID_BYTES:
            raise Error(f"comm: unique id of {_abi.COMM_ID_BYTES} bytes required")
        buf = (C.c_uint8 * _abi.COMM_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(_lib.xb_comm_create(buf, nranks, rank, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * _abi.COMM_ID_BYTES)()
        _check(_lib.xb_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def local(n: int) -> list:
        hs = (C.c_void_p * n)()
        _check(_lib.xb_comm_create_local(n, hs))
        return [Comm(_h=C.c_void_p(hs[r])) for r in range(n)]

    @property
    def size(self) -> int:
        return int(_lib.xb_comm_size(self._h))

    @property
    def rank(self) -> int:
        return int(_lib.xb_comm_rank(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.xb_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AnalogTile:
    """GPU AnalogTile (proj/include/xbarsim/tile.hpp:75-131)."""

    def __init__(self, d_out: int, d_in: int, settings: Optional[TileConfig] = None,
                 seed: int = 0, shard: Optional[tuple] = None, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            settings = settings if settings is not None else TileSettings()
            h = C.c_void_p()
            sh = None
            if shard is not None:
                sh = Shard(int(shard[0]), int(shard[1]), int(d_out), 0)
            _check(_lib.xb_tile_create(C.byref(settings), int(d_out), int(d_in),
                                       C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
                                       C.byref(sh) if sh is not None else None, C.byref(h)))
            self._h = h
        r, c, r0, rt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _lib.xb_tile_shape(self._h, C.byref(r), C.byref(c), C.byref(r0), C.byref(rt))
        self.rows, self._d_in, self.row_begin, self._d_out_total = r.value, c.value, r0.value, rt.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # (module globals are gone at interpreter exit)
            _lib.xb_tile_destroy(h)
            self._h = None

    # -- shape (tile.hpp:79-80); for a shard, d_out() is the global row count
    def d_out(self) -> int:
        return self._d_out_total

    def d_in(self) -> int:
        return self._d_in

    @property
    def handle(self):
        return self._h

    def clone(self) -> "AnalogTile":
        h = C.c_void_p()
        _check(_lib.xb_tile_clone(self._h, C.byref(h)))
        return AnalogTile(0, 0, _handle=h)

    # -- weights (tile.hpp:88-89, :103-119)
    def get_weights(self) -> np.ndarray:
        w = np.empty((self.rows, self._d_in), dtype=np.float32)
        _check(_lib.xb_tile_get_weights(self._h, _ptr(w)))
        return w

    def set_weights(self, w) -> None:
        w = np.asarray(w, dtype=np.float32)
        if w.shape != (self.rows, self._d_in):
            raise Error(f"set_weights: shape {w.shape[0]}x{w.shape[1] if w.ndim > 1 else 1}, "
                        f"expected {self.rows}x{self._d_in}")
        w = np.ascontiguousarray(w)
        _check(_lib.xb_tile_set_weights(self._h, _ptr(w)))

    def get_device(self):
        """Per-cell realization (dw_min_up, dw_min_down, w_max, w_min)."""
        arrs = [np.empty((self.rows, self._d_in), dtype=np.float32) for _ in range(4)]
        _check(_lib.xb_tile_get_device(self._h, *[_ptr(a) for a in arrs]))
        return arrs

    def set_device(self, dw_up=None, dw_down=None, w_max=None, w_min=None) -> None:
        shape = (self.rows, self._d_in)
        arrs = [None if a is None else _f32(a, shape) for a in (dw_up, dw_down, w_max, w_min)]
        _check(_lib.xb_tile_set_device(self._h, *[None if a is None else _ptr(a) for a in arrs]))

    # -- MVM (tile.hpp:82-85, :95)
    def forward(self, x, out: Optional[np.ndarray] = None) -> np.ndarray:
        """tile.hpp:80; ``out`` (float32 C-contiguous [B][d_out], e.g. in pinned
        memory) receives the result instead of a fresh array."""
        X, single = _batch(x, self._d_in, "forward")
        Y = _out(out, (X.shape[0], self.rows))
        _check(_lib.xb_tile_forward(self._h, _ptr(X), X.shape[0], _ptr(Y)))
        return Y[0] if single and out is None else Y

    def forward_with_io(self, x, io: IOParams) -> np.ndarray:
        X, single = _batch(x, self._d_in, "forward")
        Y = np.empty((X.shape[0], self.rows), dtype=np.float32)
        _check(_lib.xb_tile_forward_io(self._h, _ptr(X), X.shape[0], _ptr(Y), C.byref(io)))
        return Y[0] if single else Y

    def forward_noisy(self, x, extra_weight_sigma: float) -> np.ndarray:
        X, single = _batch(x, self._d_in, "forward")
        Y = np.empty((X.shape[0], self.rows), dtype=np.float32)
        _check(_lib.xb_tile_forward_noisy(self._h, _ptr(X), X.shape[0], _ptr(Y),
                                          float(extra_weight_sigma)))
        return Y[0] if single else Y

    def backward(self, d) -> np.ndarray:
        D, single = _batch(d, self.rows, "backward")
        G = np.empty((D.shape[0], self._d_in), dtype=np.float32)
        _check(_lib.xb_tile_backward(self._h, _ptr(D), D.shape[0], _ptr(G)))
        return G[0] if single else G

    # -- pulsed update (tile.hpp:84): B sequential updates, lr scalar or [B]
    def update(self, x, d, lr) -> None:
        X, _ = _batch(x, self._d_in, "update(x)")
        D, _ = _batch(d, self.rows, "update(d)")
        if X.shape[0] != D.shape[0]:
            raise Error("update: x and d batch sizes differ")
        lra = _lr_array(lr, X.shape[0])
        _check(_lib.xb_tile_update(self._h, _ptr(X), _ptr(D), X.shape[0],
                                   None if lra is None else lra[0]))

    def generate_trains(self, x, d, lr):
        """Packed trains the next update(x, d, lr) would draw: (xw, dw, bl)."""
        X, _ = _batch(x, self._d_in, "update(x)")
        D, _ = _batch(d, self.rows, "update(d)")
        B = X.shape[0]
        lra = _lr_array(lr, B)
        xw = np.empty((B, self._d_in), dtype=np.uint32)
        dw = np.empty((B, self.rows), dtype=np.uint32)
        bl = np.empty(B, dtype=np.int32)
        _check(_lib.xb_tile_generate_trains(self._h, _ptr(X), _ptr(D), B,
                                            None if lra is None else lra[0],
                                            xw.ctypes.data_as(_u32p), dw.ctypes.data_as(_u32p),
                                            bl.ctypes.data_as(_i32p)))
        return xw, dw, bl

    def apply_pulse_trains(self, xw, dw, flip_direction: bool = False) -> None:
        """tile.hpp:103-104 with packed uint32 trains ([B][d_in], [B][rows])."""
        xw = np.ascontiguousarray(np.atleast_2d(np.asarray(xw, dtype=np.uint32)))
        dw = np.ascontiguousarray(np.atleast_2d(np.asarray(dw, dtype=np.uint32)))
        if xw.shape[1] != self._d_in or dw.shape[1] != self.rows or xw.shape[0] != dw.shape[0]:
            raise Error("apply_coincidences: trains do not conform to tile shape")
        _check(_lib.xb_tile_apply_trains(self._h, xw.ctypes.data_as(_u32p),
                                         dw.ctypes.data_as(_u32p), xw.shape[0],
                                         int(bool(flip_direction))))

    def apply_temporal_step(self, tp: TemporalParams) -> None:
        _check(_lib.xb_tile_temporal_step(self._h, C.byref(tp)))

    def end_minibatch(self) -> None:
        _check(_lib.xb_tile_end_minibatch(self._h))

    def learning_rate(self) -> float:
        return _lib.xb_tile_learning_rate(self._h)

    def set_learning_rate(self, lr: float) -> None:
        _check(_lib.xb_tile_set_learning_rate(self._h, float(lr)))

    # -- device-resident entries (torch CUDA tensors or anything with data_ptr())
    def stream(self) -> int:
        return _lib.xb_tile_stream(self._h) or 0

    def attach_comm(self, comm: Optional["Comm"]) -> None:
        """Route this row shard's cross-shard reductions through ``comm``
        (update: max|d|; forward: BM flags; backward: max|d| and the column
        sums).  The communicator must outlive the attachment."""
        _check(_lib.xb_tile_attach_comm(self._h, comm._h if comm is not None else None))
        self._comm = comm

    def set_stream(self, stream_handle: int) -> None:
        _check(_lib.xb_tile_set_stream(self._h, C.c_void_p(stream_handle)))

    def synchronize(self) -> None:
        _check(_lib.xb_tile_synchronize(self._h))

    TIMERS = ("pulse", "trains", "forward", "backward")

    def set_timing(self, enable: bool) -> None:
        """In-stream CUDA-event timing of the kernel phases."""
        _check(_lib.xb_tile_set_timing(self._h, int(bool(enable))))

    def read_timing(self) -> dict:
        """{phase: (total_ms, launches)} since the last read (synchronises)."""
        ms = (C.c_double * 4)()
        n = (C.c_int32 * 4)()
        _check(_lib.xb_tile_read_timing(self._h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(self.TIMERS)}

    def forward_dev(self, X, Y, io: Optional[IOParams] = None, extra_sigma: float = 0.0) -> None:
        _check(_lib.xb_tile_forward_dev(self._h, _tptr(X), int(X.shape[0]), _tptr(Y),
                                        C.byref(io) if io is not None else None,
                                        float(extra_sigma)))

    def backward_dev(self, D, G) -> None:
        _check(_lib.xb_tile_backward_dev(self._h, _tptr(D), int(D.shape[0]), _tptr(G)))

    def rows_amax(self, V):
        """Device tensor [B] of max_j |V[b][j]| (on the tile's stream)."""
        import torch
        out = torch.empty(V.shape[0], dtype=torch.float32, device=V.device)
        _check(_lib.xb_rows_amax_dev(_tptr(V), int(V.shape[0]), int(V.shape[1]), _tptr(out),
                                     C.c_void_p(self.stream())))
        return out

    def backward_partial_dev(self, D, amax_d):
        """Row-shard backward phase 1: this shard's column sums [B][d_in]."""
        import torch
        P = torch.empty(D.shape[0], self._d_in, dtype=torch.float32, device=D.device)
        _check(_lib.xb_tile_backward_partial_dev(self._h, _tptr(D), int(D.shape[0]),
                                                 _tptr(amax_d), _tptr(P)))
        return P

    def backward_finish_dev(self, P, amax_d, G) -> None:
        """Row-shard backward phase 2 on the summed partials: noise, ADC, alpha."""
        _check(_lib.xb_tile_backward_finish_dev(self._h, _tptr(P), int(P.shape[0]),
                                                _tptr(amax_d), _tptr(G)))

    def update_dev(self, X, D, lr=None, amax_d=None) -> None:
        B = int(X.shape[0])
        lra = _lr_array(lr, B)
        _check(_lib.xb_tile_update_dev(self._h, _tptr(X), _tptr(D), B,
                                       None if lra is None else lra[0],
                                       None if amax_d is None else _tptr(amax_d)))

    # -- PCM inference (inference.hpp:49-70)
    def program(self, target, model: InferenceModel, seed: int) -> None:
        t = _f32(target, (self.rows, self._d_in))
        _check(_lib.xb_tile_program(self._h, _ptr(t), C.byref(model),
                                    C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF)))

    def drift_to(self, t: float) -> None:
        _check(_lib.xb_tile_drift_to(self._h, float(t)))

    def probe_readout(self, model: InferenceModel) -> float:
        out = C.c_double()
        _check(_lib.xb_tile_probe_readout(self._h, C.byref(model), C.byref(out)))
        return out.value

    def drift_compensation_factor(self, baseline: float, model: InferenceModel) -> float:
        out = C.c_double()
        _check(_lib.xb_tile_drift_compensation_factor(self._h, float(baseline), C.byref(model),
                                                      C.byref(out)))
        return out.value


def rows_amax_dev(V, out, stream: int = 0) -> None:
    _check(_lib.xb_rows_amax_dev(_tptr(V), int(V.shape[0]), int(V.shape[1]), _tptr(out),
                                 C.c_void_p(stream)))


class TransferTile:
    """GPU Tiki-Taka compound (proj/include/xbarsim/compound.hpp:93-131)."""

    def __init__(self, d_out: int, d_in: int, settings: Optional[TransferConfig] = None,
                 seed: int = 0, _handle=None):
        if _handle is not None:
            h = _handle
        else:
            settings = settings if settings is not None else TransferSettings()
            h = C.c_void_p()
            _check(_lib.xb_transfer_create(C.byref(settings), int(d_out), int(d_in),
                                           C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(h)))
        self._h = h
        self._d_out, self._d_in = int(d_out), int(d_in)
        self._fast = AnalogTile(0, 0, _handle=C.c_void_p(_lib.xb_transfer_fast(h)))
        self._slow = AnalogTile(0, 0, _handle=C.c_void_p(_lib.xb_transfer_slow(h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            # member tiles are owned by the compound
            for m in (getattr(self, "_fast", None), getattr(self, "_slow", None)):
                if m is not None:
                    m._h = None
            if _lib is not None:
                _lib.xb_transfer_destroy(h)
            self._h = None

    def d_out(self) -> int:
        return self._d_out

    def d_in(self) -> int:
        return self._d_in

    def fast_tile(self) -> AnalogTile:
        return self._fast

    def slow_tile(self) -> AnalogTile:
        return self._slow

    def forward(self, x):
        X, single = _batch(x, self._d_in, "forward")
        Y = np.empty((X.shape[0], self._d_out), dtype=np.float32)
        _check(_lib.xb_transfer_forward(self._h, _ptr(X), X.shape[0], _ptr(Y)))
        return Y[0] if single else Y

    def forward_noisy(self, x, extra_weight_sigma: float):
        """compound.cpp:228-238: both members read with the extra weight noise."""
        X, single = _batch(x, self._d_in, "forward")
        Y = np.empty((X.shape[0], self._d_out), dtype=np.float32)
        _check(_lib.xb_transfer_forward_noisy(self._h, _ptr(X), X.shape[0], _ptr(Y),
                                              float(extra_weight_sigma)))
        return Y[0] if single else Y

    def clone(self) -> "TransferTile":
        """compound.hpp:109-111: deep copy (members, RNG positions, schedule)."""
        h = C.c_void_p()
        _check(_lib.xb_transfer_clone(self._h, C.byref(h)))
        return TransferTile(self._d_out, self._d_in, _handle=h)

    def backward(self, d):
        D, single = _batch(d, self._d_out, "backward")
        G = np.empty((D.shape[0], self._d_in), dtype=np.float32)
        _check(_lib.xb_transfer_backward(self._h, _ptr(D), D.shape[0], _ptr(G)))
        return G[0] if single else G

    def update(self, x, d, lr) -> None:
        X, _ = _batch(x, self._d_in, "update(x)")
        D, _ = _batch(d, self._d_out, "update(d)")
        lra = _lr_array(lr, X.shape[0])
        _check(_lib.xb_transfer_update(self._h, _ptr(X), _ptr(D), X.shape[0],
                                       None if lra is None else lra[0]))

    def end_minibatch(self) -> None:
        _check(_lib.xb_transfer_end_minibatch(self._h))

    def transfer_step(self) -> None:
        _check(_lib.xb_transfer_step(self._h))

    def transfer_events(self) -> int:
        return int(_lib.xb_transfer_events(self._h))

    def get_weights(self) -> np.ndarray:
        w = np.empty((self._d_out, self._d_in), dtype=np.float32)
        _check(_lib.xb_transfer_get_weights(self._h, _ptr(w)))
        return w

    def set_weights(self, w) -> None:
        w = _f32(w, (self._d_out, self._d_in))
        _check(_lib.xb_transfer_set_weights(self._h, _ptr(w)))


class UnitCellTile:
    """GPU unit cell: gain-weighted device members (proj/include/xbarsim/compound.hpp:30-71)."""

    def __init__(self, d_out: int, d_in: int, settings: Optional[UnitCellConfig] = None,
                 seed: int = 0, _handle=None):
        if _handle is not None:
            h = _handle
        else:
            settings = settings if settings is not None else UnitCellSettings()
            h = C.c_void_p()
            _check(_lib.xb_unitcell_create(C.byref(settings), int(d_out), int(d_in),
                                           C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(h)))
        self._h = h
        self._d_out, self._d_in = int(d_out), int(d_in)
        self._members = []
        for k in range(_lib.xb_unitcell_n_members(h)):
            m = AnalogTile(0, 0, _handle=C.c_void_p(_lib.xb_unitcell_member(h, k)))
            self._members.append(m)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            for m in getattr(self, "_members", []):
                m._h = None  # owned by the compound
            if _lib is not None:
                _lib.xb_unitcell_destroy(h)
            self._h = None

    def d_out(self) -> int:
        return self._d_out

    def d_in(self) -> int:
        return self._d_in

    def n_members(self) -> int:
        return len(self._members)

    def member(self, k: int) -> "AnalogTile":
        """compound.hpp:53 (read-only: change members through the compound)."""
        return self._members[k]

    def clone(self) -> "UnitCellTile":
        h = C.c_void_p()
        _check(_lib.xb_unitcell_clone(self._h, C.byref(h)))
        return UnitCellTile(self._d_out, self._d_in, _handle=h)

    def forward(self, x):
        X, single = _batch(x, self._d_in, "forward")
        Y = np.empty((X.shape[0], self._d_out), dtype=np.float32)
        _check(_lib.xb_unitcell_forward(self._h, _ptr(X), X.shape[0], _ptr(Y)))
        return Y[0] if single else Y

    def forward_noisy(self, x, extra_weight_sigma: float):
        X, single = _batch(x, self._d_in, "forward")
        Y = np.empty((X.shape[0], self._d_out), dtype=np.float32)
        _check(_lib.xb_unitcell_forward_noisy(self._h, _ptr(X), X.shape[0], _ptr(Y),
                                              float(extra_weight_sigma)))
        return Y[0] if single else Y

    def backward(self, d):
        D, single = _batch(d, self._d_out, "backward")
        G = np.empty((D.shape[0], self._d_in), dtype=np.float32)
        _check(_lib.xb_unitcell_backward(self._h, _ptr(D), D.shape[0], _ptr(G)))
        return G[0] if single else G

    def update(self, x, d, lr) -> None:
        X, _ = _batch(x, self._d_in, "update(x)")
        D, _ = _batch(d, self._d_out, "update(d)")
        if X.shape[0] != D.shape[0]:
            raise Error("update: x/d lengths do not match tile shape")
        lra = _lr_array(lr, X.shape[0])
        if lra is None:
            lra = _lr_array(0.01, X.shape[0])
        _check(_lib.xb_unitcell_update(self._h, _ptr(X), _ptr(D), X.shape[0], lra[0]))

    def get_weights(self) -> np.ndarray:
        w = np.empty((self._d_out, self._d_in), dtype=np.float32)
        _check(_lib.xb_unitcell_get_weights(self._h, _ptr(w)))
        return w

    def set_weights(self, w) -> None:
        w = _f32(w, (self._d_out, self._d_in))
        _check(_lib.xb_unitcell_set_weights(self._h, _ptr(w)))

    def end_minibatch(self) -> None:
        _check(_lib.xb_unitcell_end_minibatch(self._h))

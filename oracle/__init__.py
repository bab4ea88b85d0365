"""CPU results oracle for the analog-tile hot path -- TEST INFRASTRUCTURE ONLY.

ctypes front end over the two libraries that implement ``oracle/oracle.h``:

* ``restatement``: ``oracle/liboracle.so`` built from ``xbarsim_oracle.c``, a
  plain-C restatement of the reference (``/root/reference/proj/src``); always
  available and shipped to the GPU box.
* ``reference``: ``oracle/_ref/libxbref.so`` built by ``make -C oracle ref``
  from the reference's own sources plus the ``ref_shim.cpp`` adapter; only
  present where the reference tree was available at build time.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2104_02184_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libxbref.so"),
    # the reference sources at -O2 -march=sapphirerapids: the timed reference arm
    "reference_native": os.path.join(HERE, "_ref", "libxbref_native.so"),
}
REF_TREE = "/root/reference/proj"

CONSTANT_STEP, LINEAR_STEP, SOFT_BOUNDS, EXP_STEP = 0, 1, 2, 3
NM_NONE, NM_ABS_MAX = 0, 1
PULSE_STOCHASTIC, PULSE_DETERMINISTIC = 0, 1

_d = C.c_double
_i = C.c_int32


class DeviceParams(C.Structure):
    _fields_ = [("kind", _i), ("_pad", _i), ("dw_min", _d), ("dw_min_dtod", _d),
                ("dw_min_std", _d), ("up_down", _d), ("up_down_dtod", _d), ("w_max", _d),
                ("w_min", _d), ("w_max_dtod", _d), ("w_min_dtod", _d), ("slope", _d),
                ("gamma", _d)]


class IOParams(C.Structure):
    _fields_ = [("dac_bits", _i), ("adc_bits", _i), ("input_bound", _d), ("output_bound", _d),
                ("sigma_inp", _d), ("sigma_out", _d), ("sigma_w", _d),
                ("noise_management", _i), ("is_perfect", _i)]


class UpdateParams(C.Structure):
    _fields_ = [("bl", _i), ("bl_management", _i), ("pulse_type", _i)]


class TemporalParams(C.Structure):
    _fields_ = [("decay_rate", _d), ("decay_dtod", _d), ("diffusion_sigma", _d),
                ("diffusion_dtod", _d), ("reset_prob", _d), ("reset_dtod", _d)]


class TileSettings(C.Structure):
    _fields_ = [("device", DeviceParams), ("forward_io", IOParams), ("backward_io", IOParams),
                ("update", UpdateParams), ("_pad", _i), ("temporal", TemporalParams)]


class TransferSettings(C.Structure):
    _fields_ = [("fast_device", DeviceParams), ("slow_device", DeviceParams),
                ("forward_io", IOParams), ("backward_io", IOParams), ("update", UpdateParams),
                ("_pad", _i), ("temporal", TemporalParams), ("transfer_every", _i),
                ("units_in_mbatch", _i), ("transfer_lr", _d), ("columns_per_event", _i),
                ("has_transfer_io", _i), ("gamma", _d), ("transfer_io", IOParams)]


MAX_CELL_DEVICES = 8
UC_ROUND_ROBIN, UC_ALL_TOGETHER = 0, 1


class UnitCellSettings(C.Structure):
    _fields_ = [("n_devices", _i), ("policy", _i), ("devices", DeviceParams * MAX_CELL_DEVICES),
                ("gains", _d * MAX_CELL_DEVICES), ("forward_io", IOParams),
                ("backward_io", IOParams), ("update", UpdateParams), ("_pad", _i),
                ("temporal", TemporalParams)]


class InferenceModel(C.Structure):
    _fields_ = [("prog_noise_scale", _d), ("prog_c0", _d), ("prog_c1", _d), ("prog_c2", _d),
                ("read_noise_scale", _d), ("nu_mean", _d), ("nu_std", _d), ("t0", _d),
                ("nu_min", _d), ("nu_max", _d), ("compensation_probes", _i), ("_pad", _i)]


class OracleError(RuntimeError):
    """Mirror of xbarsim::Error raised by the oracle."""


def build(reference: bool = True) -> None:
    """Compile the restatement (and, when the reference tree exists, _ref)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if reference and os.path.isdir(REF_TREE):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def available(impl: str) -> bool:
    if impl == "reference_native" and not _cpu_has("avx512f", "avx512_fp16"):
        return False  # built for sapphirerapids: never run it on an older ISA
    return os.path.exists(LIBS[impl])


def _cpu_has(*flags) -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            have = set(f.read().split())
    except OSError:
        return False
    return all(x in have for x in flags)


_P = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class Oracle:
    """One loaded oracle implementation."""

    def __init__(self, impl: str = "restatement"):
        path = LIBS[impl]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} missing; run oracle.build()")
        self.impl = impl
        L = self.lib = C.CDLL(path)
        sig = {
            "or_last_error": (C.c_char_p, []),
            "or_impl_name": (C.c_char_p, []),
            "or_device_preset": (C.c_int, [C.c_char_p, C.POINTER(DeviceParams)]),
            "or_rng_new": (_P, [C.c_uint64]),
            "or_rng_derive": (_P, [_P, C.c_char_p]),
            "or_rng_derive_idx": (_P, [_P, C.c_char_p, C.c_uint64]),
            "or_rng_free": (None, [_P]),
            "or_rng_base_seed": (C.c_uint64, [_P]),
            "or_rng_next_u64": (C.c_uint64, [_P]),
            "or_rng_uniform": (C.c_double, [_P]),
            "or_rng_gauss": (C.c_double, [_P]),
            "or_rng_bernoulli": (C.c_int, [_P, C.c_double]),
            "or_quantize_uniform": (C.c_double, [C.c_double, C.c_double, C.c_int]),
            "or_with_extra_weight_noise": (None, [C.POINTER(IOParams), C.c_double,
                                                  C.POINTER(IOParams)]),
            "or_analog_matvec": (C.c_int, [_dp, C.c_int, C.c_int, _dp, C.POINTER(IOParams), _P,
                                           C.c_int, _dp]),
            "or_realize_cell": (C.c_int, [C.POINTER(DeviceParams), _P, _dp]),
            "or_apply_pulse": (C.c_double, [_dp, C.c_double, C.c_int, C.c_int, C.c_double, _P]),
            "or_translate": (C.c_int, [_dp, C.c_int, _dp, C.c_int, C.c_double, C.c_double,
                                       C.POINTER(UpdateParams), _ip, _dp, _dp, _ip, _ip]),
            "or_generate_trains": (C.c_int, [C.c_int, _dp, C.c_int, _dp, C.c_int, _P, _u8p,
                                             _u8p]),
            "or_tile_new": (_P, [C.c_int, C.c_int, C.POINTER(TileSettings), C.c_uint64]),
            "or_tile_clone": (_P, [_P]),
            "or_tile_free": (None, [_P]),
            "or_tile_forward": (C.c_int, [_P, _dp, _dp]),
            "or_tile_backward": (C.c_int, [_P, _dp, _dp]),
            "or_tile_update": (C.c_int, [_P, _dp, _dp, C.c_double]),
            "or_tile_forward_noisy": (C.c_int, [_P, _dp, C.c_double, _dp]),
            "or_tile_forward_with_io": (C.c_int, [_P, _dp, C.POINTER(IOParams), _dp]),
            "or_tile_get_weights": (C.c_int, [_P, _dp]),
            "or_tile_set_weights": (C.c_int, [_P, _dp]),
            "or_tile_get_device": (C.c_int, [_P, _dp, _dp, _dp, _dp]),
            "or_tile_apply_pulse_trains": (C.c_int, [_P, C.c_int, _u8p, _u8p, _ip, _ip, C.c_int]),
            "or_tile_apply_temporal_step": (C.c_int, [_P, C.POINTER(TemporalParams)]),
            "or_tile_end_minibatch": (C.c_int, [_P]),
            "or_transfer_new": (_P, [C.c_int, C.c_int, C.POINTER(TransferSettings), C.c_uint64]),
            "or_transfer_free": (None, [_P]),
            "or_transfer_forward": (C.c_int, [_P, _dp, _dp]),
            "or_transfer_backward": (C.c_int, [_P, _dp, _dp]),
            "or_transfer_update": (C.c_int, [_P, _dp, _dp, C.c_double]),
            "or_transfer_end_minibatch": (C.c_int, [_P]),
            "or_transfer_step": (C.c_int, [_P]),
            "or_transfer_get_weights": (C.c_int, [_P, _dp]),
            "or_transfer_set_weights": (C.c_int, [_P, _dp]),
            "or_transfer_events": (C.c_long, [_P]),
            "or_unitcell_new": (_P, [C.c_int, C.c_int, C.POINTER(UnitCellSettings), C.c_uint64]),
            "or_unitcell_clone": (_P, [_P]),
            "or_unitcell_free": (None, [_P]),
            "or_unitcell_forward": (C.c_int, [_P, _dp, _dp]),
            "or_unitcell_backward": (C.c_int, [_P, _dp, _dp]),
            "or_unitcell_forward_noisy": (C.c_int, [_P, _dp, C.c_double, _dp]),
            "or_unitcell_update": (C.c_int, [_P, _dp, _dp, C.c_double]),
            "or_unitcell_get_weights": (C.c_int, [_P, _dp]),
            "or_unitcell_set_weights": (C.c_int, [_P, _dp]),
            "or_unitcell_end_minibatch": (C.c_int, [_P]),
            "or_unitcell_n_members": (C.c_int, [_P]),
            "or_unitcell_member": (_P, [_P, C.c_int]),
            "or_transfer_fast": (_P, [_P]),
            "or_transfer_slow": (_P, [_P]),
            "or_program": (C.c_int, [_P, _dp, C.POINTER(InferenceModel), _P, _dp, _dp]),
            "or_drift_to": (C.c_int, [_P, _dp, _dp, C.c_double, C.c_double]),
            "or_probe_readout": (C.c_int, [_P, C.POINTER(InferenceModel), _dp]),
            "or_drift_compensation_factor": (C.c_int, [_P, C.c_double, C.POINTER(InferenceModel),
                                                       _dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        for name in ("or_default_device", "or_default_io", "or_perfect_io", "or_default_update",
                     "or_default_temporal", "or_default_tile_settings",
                     "or_default_transfer_settings", "or_default_inference_model",
                     "or_default_unitcell_settings"):
            getattr(L, name).restype = None

    # ---------------------------------------------------------------- helpers
    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.or_last_error().decode())

    def default(self, kind: str):
        cls, fn = {
            "device": (DeviceParams, "or_default_device"),
            "io": (IOParams, "or_default_io"),
            "perfect_io": (IOParams, "or_perfect_io"),
            "update": (UpdateParams, "or_default_update"),
            "temporal": (TemporalParams, "or_default_temporal"),
            "tile": (TileSettings, "or_default_tile_settings"),
            "transfer": (TransferSettings, "or_default_transfer_settings"),
            "unitcell": (UnitCellSettings, "or_default_unitcell_settings"),
            "inference": (InferenceModel, "or_default_inference_model"),
        }[kind]
        obj = cls()
        getattr(self.lib, fn)(C.byref(obj))
        return obj

    def preset(self, name: str) -> DeviceParams:
        p = DeviceParams()
        self._check(self.lib.or_device_preset(name.encode(), C.byref(p)))
        return p

    def quantize(self, v, bound, bits):
        return self.lib.or_quantize_uniform(float(v), float(bound), int(bits))

    def rng(self, seed: int) -> "Rng":
        return Rng(self, self.lib.or_rng_new(C.c_uint64(seed)))

    def analog_matvec(self, w, x, io, rng: "Rng", transposed=False):
        w = _f64(w)
        x = _f64(x)
        rows, cols = w.shape
        out = np.zeros(rows if not transposed else cols)
        self._check(self.lib.or_analog_matvec(_dptr(w), rows, cols, _dptr(x), C.byref(io),
                                              rng.h, int(transposed), _dptr(out)))
        return out

    def translate(self, x, d, lr, dw_min, up):
        x = _f64(x)
        d = _f64(d)
        px = np.zeros(len(x))
        pd = np.zeros(len(d))
        sx = np.zeros(len(x), dtype=np.int32)
        sd = np.zeros(len(d), dtype=np.int32)
        bl = C.c_int()
        self._check(self.lib.or_translate(
            _dptr(x), len(x), _dptr(d), len(d), lr, dw_min, C.byref(up), C.byref(bl), _dptr(px),
            _dptr(pd), sx.ctypes.data_as(_ip), sd.ctypes.data_as(_ip)))
        return bl.value, px, pd, sx, sd

    def generate_trains(self, bl, px, pd, rng: "Rng"):
        px = _f64(px)
        pd = _f64(pd)
        xb = np.zeros((bl, len(px)), dtype=np.uint8)
        db = np.zeros((bl, len(pd)), dtype=np.uint8)
        self._check(self.lib.or_generate_trains(bl, _dptr(px), len(px), _dptr(pd), len(pd), rng.h,
                                                xb.ctypes.data_as(_u8p), db.ctypes.data_as(_u8p)))
        return xb, db

    def tile(self, d_out, d_in, settings, seed) -> "Tile":
        h = self.lib.or_tile_new(d_out, d_in, C.byref(settings), C.c_uint64(seed))
        if not h:
            raise OracleError(self.lib.or_last_error().decode())
        return Tile(self, h, d_out, d_in, own=True)

    def unitcell(self, d_out, d_in, settings, seed) -> "UnitCell":
        h = self.lib.or_unitcell_new(d_out, d_in, C.byref(settings), C.c_uint64(seed))
        if not h:
            raise OracleError(self.lib.or_last_error().decode())
        return UnitCell(self, h, d_out, d_in)

    def transfer(self, d_out, d_in, settings, seed) -> "Transfer":
        h = self.lib.or_transfer_new(d_out, d_in, C.byref(settings), C.c_uint64(seed))
        if not h:
            raise OracleError(self.lib.or_last_error().decode())
        return Transfer(self, h, d_out, d_in)


class Rng:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.lib.or_rng_free(self.h)
        except Exception:
            pass

    def derive(self, name: str, index=None) -> "Rng":
        if index is None:
            return Rng(self.o, self.o.lib.or_rng_derive(self.h, name.encode()))
        return Rng(self.o, self.o.lib.or_rng_derive_idx(self.h, name.encode(),
                                                        C.c_uint64(index)))

    def base_seed(self) -> int:
        return self.o.lib.or_rng_base_seed(self.h)

    def next_u64(self) -> int:
        return self.o.lib.or_rng_next_u64(self.h)

    def uniform(self) -> float:
        return self.o.lib.or_rng_uniform(self.h)

    def gauss(self) -> float:
        return self.o.lib.or_rng_gauss(self.h)

    def bernoulli(self, p) -> bool:
        return bool(self.o.lib.or_rng_bernoulli(self.h, float(p)))


class Tile:
    """Oracle AnalogTile (proj/include/xbarsim/tile.hpp:75-131)."""

    def __init__(self, o: Oracle, h, d_out, d_in, own=True):
        self.o, self.h, self.d_out, self.d_in, self.own = o, h, d_out, d_in, own

    def __del__(self):
        if self.own:
            try:
                self.o.lib.or_tile_free(self.h)
            except Exception:
                pass

    def clone(self) -> "Tile":
        return Tile(self.o, self.o.lib.or_tile_clone(self.h), self.d_out, self.d_in)

    def forward(self, x):
        x = _f64(x)
        assert x.shape == (self.d_in,)
        y = np.zeros(self.d_out)
        self.o._check(self.o.lib.or_tile_forward(self.h, _dptr(x), _dptr(y)))
        return y

    def backward(self, d):
        d = _f64(d)
        assert d.shape == (self.d_out,)
        g = np.zeros(self.d_in)
        self.o._check(self.o.lib.or_tile_backward(self.h, _dptr(d), _dptr(g)))
        return g

    def forward_noisy(self, x, extra):
        x = _f64(x)
        y = np.zeros(self.d_out)
        self.o._check(self.o.lib.or_tile_forward_noisy(self.h, _dptr(x), extra, _dptr(y)))
        return y

    def forward_with_io(self, x, io):
        x = _f64(x)
        y = np.zeros(self.d_out)
        self.o._check(self.o.lib.or_tile_forward_with_io(self.h, _dptr(x), C.byref(io), _dptr(y)))
        return y

    def update(self, x, d, lr):
        x = _f64(x)
        d = _f64(d)
        assert x.shape == (self.d_in,) and d.shape == (self.d_out,)
        self.o._check(self.o.lib.or_tile_update(self.h, _dptr(x), _dptr(d), float(lr)))

    def get_weights(self):
        w = np.zeros((self.d_out, self.d_in))
        self.o._check(self.o.lib.or_tile_get_weights(self.h, _dptr(w)))
        return w

    def set_weights(self, w):
        w = _f64(w)
        assert w.shape == (self.d_out, self.d_in)
        self.o._check(self.o.lib.or_tile_set_weights(self.h, _dptr(w)))

    def get_device(self):
        arrs = [np.zeros((self.d_out, self.d_in)) for _ in range(4)]
        self.o._check(self.o.lib.or_tile_get_device(self.h, *[_dptr(a) for a in arrs]))
        return arrs  # dw_up, dw_down, w_max, w_min

    def apply_pulse_trains(self, bl, xbits, dbits, sign_x, sign_d, flip=False):
        xb = np.ascontiguousarray(xbits, dtype=np.uint8)
        db = np.ascontiguousarray(dbits, dtype=np.uint8)
        sx = np.ascontiguousarray(sign_x, dtype=np.int32)
        sd = np.ascontiguousarray(sign_d, dtype=np.int32)
        assert xb.shape == (bl, self.d_in) and db.shape == (bl, self.d_out)
        self.o._check(self.o.lib.or_tile_apply_pulse_trains(
            self.h, bl, xb.ctypes.data_as(_u8p), db.ctypes.data_as(_u8p), sx.ctypes.data_as(_ip),
            sd.ctypes.data_as(_ip), int(flip)))

    def apply_temporal_step(self, tp):
        self.o._check(self.o.lib.or_tile_apply_temporal_step(self.h, C.byref(tp)))

    def end_minibatch(self):
        self.o._check(self.o.lib.or_tile_end_minibatch(self.h))

    # PCM inference (proj/src/inference.cpp:34-110)
    def program(self, target, model, rng: Rng):
        target = _f64(target)
        w0 = np.zeros((self.d_out, self.d_in))
        nu = np.zeros((self.d_out, self.d_in))
        self.o._check(self.o.lib.or_program(self.h, _dptr(target), C.byref(model), rng.h,
                                            _dptr(w0), _dptr(nu)))
        return w0, nu

    def drift_to(self, w0, nu, t0, t):
        w0 = _f64(w0)
        nu = _f64(nu)
        self.o._check(self.o.lib.or_drift_to(self.h, _dptr(w0), _dptr(nu), t0, t))

    def probe_readout(self, model):
        out = C.c_double()
        self.o._check(self.o.lib.or_probe_readout(self.h, C.byref(model), C.byref(out)))
        return out.value

    def drift_compensation_factor(self, baseline, model):
        out = C.c_double()
        self.o._check(self.o.lib.or_drift_compensation_factor(self.h, baseline, C.byref(model),
                                                              C.byref(out)))
        return out.value


class Transfer:
    """Oracle TransferTile (proj/include/xbarsim/compound.hpp:93-131)."""

    def __init__(self, o: Oracle, h, d_out, d_in):
        self.o, self.h, self.d_out, self.d_in = o, h, d_out, d_in
        self.fast = Tile(o, o.lib.or_transfer_fast(h), d_out, d_in, own=False)
        self.slow = Tile(o, o.lib.or_transfer_slow(h), d_out, d_in, own=False)

    def __del__(self):
        try:
            self.o.lib.or_transfer_free(self.h)
        except Exception:
            pass

    def forward(self, x):
        x = _f64(x)
        y = np.zeros(self.d_out)
        self.o._check(self.o.lib.or_transfer_forward(self.h, _dptr(x), _dptr(y)))
        return y

    def backward(self, d):
        d = _f64(d)
        g = np.zeros(self.d_in)
        self.o._check(self.o.lib.or_transfer_backward(self.h, _dptr(d), _dptr(g)))
        return g

    def update(self, x, d, lr):
        x = _f64(x)
        d = _f64(d)
        self.o._check(self.o.lib.or_transfer_update(self.h, _dptr(x), _dptr(d), float(lr)))

    def end_minibatch(self):
        self.o._check(self.o.lib.or_transfer_end_minibatch(self.h))

    def transfer_step(self):
        self.o._check(self.o.lib.or_transfer_step(self.h))

    def get_weights(self):
        w = np.zeros((self.d_out, self.d_in))
        self.o._check(self.o.lib.or_transfer_get_weights(self.h, _dptr(w)))
        return w

    def set_weights(self, w):
        w = _f64(w)
        self.o._check(self.o.lib.or_transfer_set_weights(self.h, _dptr(w)))

    def events(self) -> int:
        return self.o.lib.or_transfer_events(self.h)


class UnitCell:
    """Oracle UnitCellTile (proj/include/xbarsim/compound.hpp:30-71)."""

    def __init__(self, o: Oracle, h, d_out, d_in):
        self.o, self.h, self.d_out, self.d_in = o, h, d_out, d_in
        self.members = [Tile(o, o.lib.or_unitcell_member(h, k), d_out, d_in, own=False)
                        for k in range(o.lib.or_unitcell_n_members(h))]

    def __del__(self):
        try:
            self.o.lib.or_unitcell_free(self.h)
        except Exception:
            pass

    def clone(self) -> "UnitCell":
        return UnitCell(self.o, self.o.lib.or_unitcell_clone(self.h), self.d_out, self.d_in)

    def forward(self, x):
        x = _f64(x)
        y = np.zeros(self.d_out)
        self.o._check(self.o.lib.or_unitcell_forward(self.h, _dptr(x), _dptr(y)))
        return y

    def forward_noisy(self, x, extra):
        x = _f64(x)
        y = np.zeros(self.d_out)
        self.o._check(self.o.lib.or_unitcell_forward_noisy(self.h, _dptr(x), float(extra),
                                                           _dptr(y)))
        return y

    def backward(self, d):
        d = _f64(d)
        g = np.zeros(self.d_in)
        self.o._check(self.o.lib.or_unitcell_backward(self.h, _dptr(d), _dptr(g)))
        return g

    def update(self, x, d, lr):
        x = _f64(x)
        d = _f64(d)
        self.o._check(self.o.lib.or_unitcell_update(self.h, _dptr(x), _dptr(d), float(lr)))

    def end_minibatch(self):
        self.o._check(self.o.lib.or_unitcell_end_minibatch(self.h))

    def get_weights(self):
        w = np.zeros((self.d_out, self.d_in))
        self.o._check(self.o.lib.or_unitcell_get_weights(self.h, _dptr(w)))
        return w

    def set_weights(self, w):
        w = _f64(w)
        self.o._check(self.o.lib.or_unitcell_set_weights(self.h, _dptr(w)))


_cache: dict[str, Oracle] = {}


def load(impl: str = "restatement") -> Oracle:
    if impl not in _cache:
        _cache[impl] = Oracle(impl)
    return _cache[impl]

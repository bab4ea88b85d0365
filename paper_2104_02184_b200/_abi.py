"""ctypes binding of the C ABI in include/xbtile.h (libxbtile.so).

The library is loaded from the package directory (built in-tree by
``paper_2104_02184_b200.build``).  There is no fallback: if the shared
object is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# XBTILE_LIB selects an experiment build (paper_2104_02184_b200/build.py --out=...)
LIB_PATH = os.environ.get("XBTILE_LIB") or os.path.join(PKG, "libxbtile.so")

CONSTANT_STEP, LINEAR_STEP, SOFT_BOUNDS, EXP_STEP = 0, 1, 2, 3
NM_NONE, NM_ABS_MAX = 0, 1
BM_NONE, BM_ITERATIVE = 0, 1
PULSE_STOCHASTIC, PULSE_DETERMINISTIC = 0, 1
MVM_FP32, MVM_TF32, MVM_TF32X3 = 0, 1, 2
W_AUTO, W_FP32, W_FP32X2 = 0, 1, 2

_d = C.c_double
_i = C.c_int32


class DeviceParams(C.Structure):
    """proj/include/xbarsim/device.hpp:24-39."""
    _fields_ = [("kind", _i), ("_pad", _i), ("dw_min", _d), ("dw_min_dtod", _d),
                ("dw_min_std", _d), ("up_down", _d), ("up_down_dtod", _d), ("w_max", _d),
                ("w_min", _d), ("w_max_dtod", _d), ("w_min_dtod", _d), ("slope", _d),
                ("gamma", _d)]


class IOParams(C.Structure):
    """proj/include/xbarsim/io.hpp:21-33 (+ bound management)."""
    _fields_ = [("dac_bits", _i), ("adc_bits", _i), ("input_bound", _d), ("output_bound", _d),
                ("sigma_inp", _d), ("sigma_out", _d), ("sigma_w", _d),
                ("noise_management", _i), ("is_perfect", _i), ("bound_management", _i),
                ("bm_max_iter", _i)]


class UpdateParams(C.Structure):
    """proj/include/xbarsim/pulsed.hpp:21-27."""
    _fields_ = [("bl", _i), ("bl_management", _i), ("pulse_type", _i)]


class TemporalParams(C.Structure):
    """proj/include/xbarsim/tile.hpp:24-36."""
    _fields_ = [("decay_rate", _d), ("decay_dtod", _d), ("diffusion_sigma", _d),
                ("diffusion_dtod", _d), ("reset_prob", _d), ("reset_dtod", _d)]


class TileConfig(C.Structure):
    """proj/include/xbarsim/tile.hpp:38-44 (TileSettings) + mvm_precision, weight_precision."""
    _fields_ = [("device", DeviceParams), ("forward_io", IOParams), ("backward_io", IOParams),
                ("update", UpdateParams), ("mvm_precision", _i), ("temporal", TemporalParams),
                ("weight_precision", _i), ("_pad2", _i)]


class Shard(C.Structure):
    _fields_ = [("row_begin", _i), ("row_end", _i), ("d_out_total", _i), ("_pad", _i)]


class InferenceModel(C.Structure):
    """proj/include/xbarsim/inference.hpp:21-36."""
    _fields_ = [("prog_noise_scale", _d), ("prog_c0", _d), ("prog_c1", _d), ("prog_c2", _d),
                ("read_noise_scale", _d), ("nu_mean", _d), ("nu_std", _d), ("t0", _d),
                ("nu_min", _d), ("nu_max", _d), ("compensation_probes", _i), ("_pad", _i)]


class TransferConfig(C.Structure):
    """proj/include/xbarsim/compound.hpp:76-91."""
    _fields_ = [("fast_device", DeviceParams), ("slow_device", DeviceParams),
                ("forward_io", IOParams), ("backward_io", IOParams), ("update", UpdateParams),
                ("mvm_precision", _i), ("temporal", TemporalParams), ("transfer_every", _i),
                ("units_in_mbatch", _i), ("transfer_lr", _d), ("columns_per_event", _i),
                ("has_transfer_io", _i), ("gamma", _d), ("transfer_io", IOParams)]


MAX_CELL_DEVICES = 8
UC_ROUND_ROBIN, UC_ALL_TOGETHER = 0, 1


class UnitCellConfig(C.Structure):
    """proj/include/xbarsim/compound.hpp:15-28 (fixed arrays of n_devices <= 8)."""
    _fields_ = [("n_devices", _i), ("policy", _i), ("devices", DeviceParams * MAX_CELL_DEVICES),
                ("gains", _d * MAX_CELL_DEVICES), ("forward_io", IOParams),
                ("backward_io", IOParams), ("update", UpdateParams), ("mvm_precision", _i),
                ("temporal", TemporalParams)]


_P = C.c_void_p
_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)

# name -> (restype, argtypes): exactly the declarations of include/xbtile.h
SIGNATURES = {
    "xb_abi_version": (C.c_int, []),
    "xb_last_error": (C.c_char_p, []),
    "xb_device_check": (C.c_int, []),
    "xb_launch_count": (C.c_uint64, []),
    "xb_launch_floor_us": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "xb_default_device": (None, [C.POINTER(DeviceParams)]),
    "xb_default_io": (None, [C.POINTER(IOParams)]),
    "xb_perfect_io": (None, [C.POINTER(IOParams)]),
    "xb_default_config": (None, [C.POINTER(TileConfig)]),
    "xb_default_transfer_config": (None, [C.POINTER(TransferConfig)]),
    "xb_default_inference_model": (None, [C.POINTER(InferenceModel)]),
    "xb_device_preset": (C.c_int, [C.c_char_p, C.POINTER(DeviceParams)]),
    "xb_tile_create": (C.c_int, [C.POINTER(TileConfig), C.c_int, C.c_int, C.c_uint64,
                                 C.POINTER(Shard), C.POINTER(_P)]),
    "xb_tile_destroy": (C.c_int, [_P]),
    "xb_tile_clone": (C.c_int, [_P, C.POINTER(_P)]),
    "xb_tile_shape": (C.c_int, [_P, _i32p, _i32p, _i32p, _i32p]),
    "xb_tile_set_stream": (C.c_int, [_P, _P]),
    "xb_tile_stream": (_P, [_P]),
    "xb_tile_set_weights": (C.c_int, [_P, _fp]),
    "xb_tile_get_weights": (C.c_int, [_P, _fp]),
    "xb_tile_set_device": (C.c_int, [_P, _fp, _fp, _fp, _fp]),
    "xb_tile_get_device": (C.c_int, [_P, _fp, _fp, _fp, _fp]),
    "xb_tile_forward": (C.c_int, [_P, _fp, C.c_int, _fp]),
    "xb_tile_forward_io": (C.c_int, [_P, _fp, C.c_int, _fp, C.POINTER(IOParams)]),
    "xb_tile_forward_noisy": (C.c_int, [_P, _fp, C.c_int, _fp, C.c_double]),
    "xb_tile_backward": (C.c_int, [_P, _fp, C.c_int, _fp]),
    "xb_tile_update": (C.c_int, [_P, _fp, _fp, C.c_int, _dp]),
    "xb_tile_apply_trains": (C.c_int, [_P, _u32p, _u32p, C.c_int, C.c_int]),
    "xb_tile_generate_trains": (C.c_int, [_P, _fp, _fp, C.c_int, _dp, _u32p, _u32p, _i32p]),
    "xb_tile_temporal_step": (C.c_int, [_P, C.POINTER(TemporalParams)]),
    "xb_tile_end_minibatch": (C.c_int, [_P]),
    "xb_tile_set_learning_rate": (C.c_int, [_P, C.c_double]),
    "xb_tile_learning_rate": (C.c_double, [_P]),
    "xb_tile_forward_dev": (C.c_int, [_P, _P, C.c_int, _P, C.POINTER(IOParams), C.c_double]),
    "xb_tile_backward_dev": (C.c_int, [_P, _P, C.c_int, _P]),
    "xb_tile_update_dev": (C.c_int, [_P, _P, _P, C.c_int, _dp, _P]),
    "xb_tile_backward_partial_dev": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "xb_tile_backward_finish_dev": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "xb_rows_amax_dev": (C.c_int, [_P, C.c_int, C.c_int, _P, _P]),
    "xb_tile_synchronize": (C.c_int, [_P]),
    "xb_tile_set_timing": (C.c_int, [_P, C.c_int]),
    "xb_tile_read_timing": (C.c_int, [_P, _dp, _i32p]),
    "xb_tile_program": (C.c_int, [_P, _fp, C.POINTER(InferenceModel), C.c_uint64]),
    "xb_tile_drift_to": (C.c_int, [_P, C.c_double]),
    "xb_tile_probe_readout": (C.c_int, [_P, C.POINTER(InferenceModel), _dp]),
    "xb_tile_drift_compensation_factor": (C.c_int, [_P, C.c_double, C.POINTER(InferenceModel),
                                                    _dp]),
    "xb_transfer_create": (C.c_int, [C.POINTER(TransferConfig), C.c_int, C.c_int, C.c_uint64,
                                     C.POINTER(_P)]),
    "xb_transfer_destroy": (C.c_int, [_P]),
    "xb_transfer_forward": (C.c_int, [_P, _fp, C.c_int, _fp]),
    "xb_transfer_backward": (C.c_int, [_P, _fp, C.c_int, _fp]),
    "xb_transfer_forward_noisy": (C.c_int, [_P, _fp, C.c_int, _fp, C.c_double]),
    "xb_transfer_clone": (C.c_int, [_P, C.POINTER(_P)]),
    "xb_transfer_update": (C.c_int, [_P, _fp, _fp, C.c_int, _dp]),
    "xb_transfer_end_minibatch": (C.c_int, [_P]),
    "xb_transfer_step": (C.c_int, [_P]),
    "xb_transfer_get_weights": (C.c_int, [_P, _fp]),
    "xb_transfer_set_weights": (C.c_int, [_P, _fp]),
    "xb_transfer_events": (C.c_long, [_P]),
    "xb_default_unitcell_config": (None, [C.POINTER(UnitCellConfig)]),
    "xb_unitcell_create": (C.c_int, [C.POINTER(UnitCellConfig), C.c_int, C.c_int, C.c_uint64,
                                     C.POINTER(_P)]),
    "xb_unitcell_destroy": (C.c_int, [_P]),
    "xb_unitcell_clone": (C.c_int, [_P, C.POINTER(_P)]),
    "xb_unitcell_forward": (C.c_int, [_P, _fp, C.c_int, _fp]),
    "xb_unitcell_forward_noisy": (C.c_int, [_P, _fp, C.c_int, _fp, C.c_double]),
    "xb_unitcell_backward": (C.c_int, [_P, _fp, C.c_int, _fp]),
    "xb_unitcell_update": (C.c_int, [_P, _fp, _fp, C.c_int, _dp]),
    "xb_unitcell_get_weights": (C.c_int, [_P, _fp]),
    "xb_unitcell_set_weights": (C.c_int, [_P, _fp]),
    "xb_unitcell_end_minibatch": (C.c_int, [_P]),
    "xb_unitcell_n_members": (C.c_int, [_P]),
    "xb_unitcell_member": (_P, [_P, C.c_int]),
    "xb_transfer_fast": (_P, [_P]),
    "xb_transfer_slow": (_P, [_P]),
    "xb_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "xb_comm_create": (C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.POINTER(_P)]),
    "xb_comm_create_local": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "xb_comm_destroy": (C.c_int, [_P]),
    "xb_comm_size": (C.c_int, [_P]),
    "xb_comm_rank": (C.c_int, [_P]),
    "xb_tile_attach_comm": (C.c_int, [_P, _P]),
}
COMM_ID_BYTES = 128


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python paper_2104_02184_b200/build.py` "
            "(there is no CPU fallback for the B200 analog tile)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.xb_abi_version() != 1:
        raise ImportError("libxbtile ABI version mismatch")
    return lib

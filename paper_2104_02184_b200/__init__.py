"""B200-native analog-tile hot path (pulsed update + noisy MVM) behind the
reference's tile API.

The compute lives in libxbtile.so (CUDA C++, sm_100a) reached through the C
ABI in include/xbtile.h; this package is the host-side mirror of the
reference interface.  Importing it without the built library raises: there
is no CPU fallback.
"""
from ._abi import (BM_ITERATIVE, BM_NONE, CONSTANT_STEP, EXP_STEP, LINEAR_STEP, MVM_FP32,
                   MVM_TF32, MVM_TF32X3, NM_ABS_MAX, NM_NONE, PULSE_DETERMINISTIC,
                   PULSE_STOCHASTIC, SOFT_BOUNDS, UC_ALL_TOGETHER, UC_ROUND_ROBIN, W_AUTO,
                   W_FP32, W_FP32X2, DeviceParams,
                   InferenceModel, IOParams, TemporalParams, TileConfig, TransferConfig,
                   UnitCellConfig, UpdateParams)
from .tile import (AnalogTile, Comm, Error, InferenceNoiseModel, TileSettings, TransferSettings,
                   TransferTile, UnitCellSettings, UnitCellTile, default_device, default_io,
                   device_check, device_preset, io_off, launch_count, launch_floor_us, perfect_io,
                   rows_amax_dev)

__all__ = [
    "AnalogTile", "TransferTile", "TileSettings", "TransferSettings", "InferenceNoiseModel",
    "DeviceParams", "IOParams", "UpdateParams", "TemporalParams", "TileConfig", "TransferConfig",
    "InferenceModel", "Error", "device_preset", "default_device", "default_io", "perfect_io",
    "io_off", "device_check", "launch_count", "launch_floor_us", "rows_amax_dev", "CONSTANT_STEP", "LINEAR_STEP",
    "SOFT_BOUNDS", "EXP_STEP", "NM_NONE", "NM_ABS_MAX", "BM_NONE", "BM_ITERATIVE",
    "PULSE_STOCHASTIC", "PULSE_DETERMINISTIC", "MVM_FP32", "MVM_TF32", "MVM_TF32X3",
    "UnitCellTile", "UnitCellSettings", "UnitCellConfig", "UC_ROUND_ROBIN", "UC_ALL_TOGETHER",
    "W_AUTO", "W_FP32", "W_FP32X2", "Comm",
]

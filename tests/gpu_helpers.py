"""Shared helpers for the -m gpu parity tests (GPU path vs the CPU oracle)."""
from __future__ import annotations

import numpy as np

import oracle
import paper_2104_02184_b200 as xb
from paper_2104_02184_b200 import trains as T


def oracle_settings(O, gpu_cfg):
    """Mirror a GPU TileConfig into the oracle's TileSettings."""
    s = O.default("tile")
    for f in ("kind", "dw_min", "dw_min_dtod", "dw_min_std", "up_down", "up_down_dtod", "w_max",
              "w_min", "w_max_dtod", "w_min_dtod", "slope", "gamma"):
        setattr(s.device, f, getattr(gpu_cfg.device, f))
    for side in ("forward_io", "backward_io"):
        src, dst = getattr(gpu_cfg, side), getattr(s, side)
        for f in ("dac_bits", "adc_bits", "input_bound", "output_bound", "sigma_inp", "sigma_out",
                  "sigma_w", "noise_management", "is_perfect"):
            setattr(dst, f, getattr(src, f))
    s.update.bl = gpu_cfg.update.bl
    s.update.bl_management = gpu_cfg.update.bl_management
    s.update.pulse_type = gpu_cfg.update.pulse_type
    return s


def oracle_io(O, io):
    o = O.default("io")
    for f in ("dac_bits", "adc_bits", "input_bound", "output_bound", "sigma_inp", "sigma_out",
              "sigma_w", "noise_management", "is_perfect"):
        setattr(o, f, getattr(io, f))
    return o


def twin(cfg, d_out, d_in, seed=1, w_scale=0.1, w_seed=3):
    """A GPU tile and an oracle tile with the SAME realization and weights.

    The GPU realization is replaced by the oracle's (fp64 -> fp32), the
    protocol of SURVEY.md 8c(iv)."""
    O = oracle.load("restatement")
    g = xb.AnalogTile(d_out, d_in, cfg, seed)
    o = O.tile(d_out, d_in, oracle_settings(O, cfg), seed)
    up, dn, wmax, wmin = o.get_device()
    g.set_device(up, dn, wmax, wmin)
    # give the oracle the fp32-rounded realization too, so both act on identical cells
    w0 = np.random.default_rng(w_seed).uniform(-w_scale, w_scale, (d_out, d_in)).astype(np.float32)
    g.set_weights(w0)
    o.set_weights(w0.astype(np.float64))
    return g, o


def apply_words_to_oracle(o, xw, dw, bl, flip=False):
    """Feed GPU-packed trains, sample by sample, to the oracle tile."""
    for b in range(xw.shape[0]):
        nb = int(bl[b]) if np.ndim(bl) else int(bl)
        if nb <= 0:
            continue
        xb_bits, sx = T.unpack(xw[b], nb)
        db_bits, sd = T.unpack(dw[b], nb)
        # a zero line carries no bits; its sign is irrelevant for counting
        o.apply_pulse_trains(nb, xb_bits, db_bits, sx, sd, flip=flip)


def close(a, b, rtol, floor):
    """|a - b| <= rtol * max(|b|, floor) elementwise (the reference's
    tol * max(1, |y|) form, proj/tests/test_tile.cpp:263)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) <= rtol * np.maximum(np.abs(b), floor)

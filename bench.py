"""Headline benchmark: pulsed-update cell-updates/s and noisy-MVM samples/s on
a 4096 x 4096 SoftBounds (reram_sb) tile, BL = 31, batch 256 (BASELINE.json
north star).  One step = one mini-batch through the tile: the noisy forward of
256 samples (default IO: DAC 7 b, ADC 9 b, sigma_out 0.06, abs-max, bound
management on) followed by the 256 sequential pulsed updates.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one process per GPU): the north star's multi-GPU case,
BASELINE config 5 -- ONE logical 16384 x 16384 reram_sb tile row-sharded over
the N GPUs (strong scaling; 16384/N rows per GPU), the same step (forward
with output noise, bound management and ADC, then the pulsed update of 256
samples).  The cross-GPU reductions (max|d| for translate, the bound-
management flags) run inside libxbtile over NCCL (xb_comm, NVLink/NVSwitch);
torch.distributed (gloo) only bootstraps the NCCL id and gathers the timings.
The line also carries a weak-scaling measurement ((4096 N) x 4096, 4096 rows
per GPU) and the PCM program + drift_to pass on the 16384^2 shards.

--impl reference times the reference CPU implementation (oracle/_ref, the
xbarsim sources compiled here; the C restatement when _ref is absent) on the
host cores, the same per-sample work per step, one independent tile per core.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ROWS = 4096  # rows per GPU
N_COLS = 4096
BATCH = 256
LR = 0.01
METRIC = "pulsed-update cell-updates/s (4096x4096 reram_sb tile, BL=31, batch 256; " \
         "step = noisy forward + pulsed update)"
UNIT = "cell-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ============================================================ our arm
CFG5 = 16384  # BASELINE config 5: 16384 x 16384 tile, row-sharded over N GPUs


def tile_settings(xb, prec=None):
    dev = xb.device_preset("reram_sb")
    fwd = xb.default_io()
    fwd.bound_management = xb.BM_ITERATIVE
    fwd.bm_max_iter = 10
    # TF32 tensor-core contraction: its ~1e-3 relative error (of the dot-product
    # scale) is far below sigma_out = 0.06 and the 9-bit ADC step
    cfg = xb.TileSettings(device=dev, forward_io=fwd, backward_io=xb.default_io(),
                          mvm_precision=prec if prec is not None else xb.MVM_TF32)
    cfg.update.bl = 31
    return cfg


def make_tile(xb, rank, world, d_out=N_ROWS, d_in=N_COLS, comm=None):
    """This rank's shard of a d_out x d_in tile (the whole tile when world == 1)."""
    from paper_2104_02184_b200.parallel import partition_rows
    cfg = tile_settings(xb)
    if world == 1:
        return xb.AnalogTile(d_out, d_in, cfg, 1234), cfg, (0, d_out)
    r0, r1 = partition_rows(d_out, world, rank)
    t = xb.AnalogTile(d_out, d_in, cfg, 1234, shard=(r0, r1))
    t.attach_comm(comm)
    return t, cfg, (r0, r1)


def timed_steps(torch, dist, tile, stream, Xs, Ds, Y, steps, warmup, world, clk=None):
    """W untimed steps, then K steps between CUDA events on the tile stream,
    bracketed by a barrier + device sync; returns the max over ranks (ms)
    plus this rank's phase timings."""
    def step(s):
        tile.forward_dev(Xs[s], Y)        # sharded: BM flags all-reduced per pass (NCCL)
        tile.update_dev(Xs[s], Ds[s], LR)  # sharded: global max|d| all-reduced (NCCL)
    for s in range(warmup):
        step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tile.set_timing(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(steps):
        step(warmup + s)
    e1.record(stream)
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__(None, None, None)
    timing = tile.read_timing()
    tile.set_timing(False)
    t = torch.tensor([e0.elapsed_time(e1)] + [timing[k][0] for k in tile.TIMERS[:3]],
                     dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # gloo, CPU tensor
    return t.tolist(), [timing[k][1] for k in tile.TIMERS]


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2104_02184_b200 as xb
    from paper_2104_02184_b200.parallel import nccl_comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # validation-only override (never for a reported number): every rank on one
    # device, loopback collectives instead of NCCL (tests/test_gpu_bench.py)
    loopback = bool(os.environ.get("XB_BENCH_DEVICE"))
    if loopback:
        local = int(os.environ["XB_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        # gloo: bootstrap (NCCL id) and timing gathers only; data path = libxbtile + NCCL
        dist.init_process_group("gloo")
        comm = loopback_comm(xb, dist, world, rank) if loopback else nccl_comm()
    dev = torch.device("cuda", local)
    # a dedicated (non-default) stream shared by torch and the tile, so CUDA
    # events and the tile's kernels (and its NCCL calls) are ordered on one queue
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    R_total = N_ROWS if world == 1 else CFG5
    C = N_COLS if world == 1 else CFG5
    tile, cfg, (r0, r1) = make_tile(xb, rank, world, R_total, C, comm)
    tile.set_stream(stream.cuda_stream)
    rows = r1 - r0
    g = torch.Generator(device=dev)
    g.manual_seed(7 + rank)
    w0 = torch.rand(rows, C, generator=g, device=dev) * 0.2 - 0.1
    tile.set_weights(w0.cpu().numpy())
    nsets = args.steps + args.warmup
    # distinct synthetic batches per step; x is replicated (same seed on every rank)
    gx = torch.Generator(device=dev)
    gx.manual_seed(7)
    nx = min(nsets, 8) if world > 1 else nsets  # 16 MB per x batch at 16384 columns
    Xs = [torch.rand(BATCH, C, generator=gx, device=dev) * 2 - 1 for _ in range(nx)]
    Ds = [torch.rand(BATCH, rows, generator=g, device=dev) * 2 - 1 for _ in range(nx)]
    Xs = [Xs[k % nx] for k in range(nsets)]
    Ds = [Ds[k % nx] for k in range(nsets)]
    Y = torch.empty(BATCH, rows, device=dev)

    clk = Clocks(local).__enter__()  # sampling starts before the warm-up so it spans the timed region
    launches0 = xb.launch_count()
    (ms_total, ms_pulse, ms_trains, ms_fwd), ph_n = timed_steps(
        torch, dist, tile, stream, Xs, Ds, Y, args.steps, args.warmup, world, clk)
    launches = xb.launch_count() - launches0
    launches = int(round(launches * args.steps / (args.steps + args.warmup)))  # timed steps only
    ms_step = ms_total / args.steps
    cells = float(R_total) * C * BATCH
    value = cells / (ms_step * 1e-3)

    # ---------- e2e through the public host-buffer API (pinned host inputs)
    n_e2e = max(2, min(args.steps, 10))
    Xh = [Xs[k].cpu().pin_memory().numpy() for k in range(n_e2e)]
    Dh = [Ds[k].cpu().pin_memory().numpy() for k in range(n_e2e)]
    e2e_tile, _, _ = make_tile(xb, rank, world, R_total, C, comm)
    e2e_tile.set_weights(w0.cpu().numpy())
    # the result lands in pinned host memory (DMA at full PCIe rate)
    yh = torch.empty(BATCH, rows, dtype=torch.float32).pin_memory().numpy()
    for k in range(2):  # warm
        e2e_tile.forward(Xh[k], out=yh)
        e2e_tile.update(Xh[k], Dh[k], LR)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(n_e2e):
        e2e_tile.forward(Xh[k], out=yh)
        e2e_tile.update(Xh[k], Dh[k], LR)
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    _ = float(yh[0, 0])
    del e2e_tile
    e2e = {"value": cells * n_e2e / float(el.item()), "unit": UNIT,
           "h2d_bytes_per_step": int(world * (BATCH * C * 4 * 2 + BATCH * rows * 4)),
           "d2h_bytes_per_step": int(world * BATCH * rows * 4),
           "steps": n_e2e,
           "api": ("AnalogTile.forward(X host) + AnalogTile.update(X, D host)" if world == 1 else
                   "per rank: AnalogTile(shard).forward(X host) + update(X, D_local host), "
                   "NCCL reductions inside libxbtile")}

    extra = {}
    if world > 1:
        extra = sharded_extras(torch, dist, xb, tile, comm, stream, rank, world, r0, r1, args)

    if rank == 0:
        pk, pk_kind = peaks()
        clocks = clk.summary()
        # --- measured pulses per cell-update (k-bar) on 32 samples of the workload:
        # sum_ij popc(x_j & d_i) = sum_t (#x lines firing slot t)(#d lines firing slot t)
        kbar = measure_kbar(xb, R_total if world == 1 else rows, C, Xs[0][:32].cpu().numpy(),
                            Ds[0][:32].cpu().numpy())
        # --- roofline of the dominant kernel (pulse_kernel): integer pipe, SURVEY 8d
        int_ops = (2.0 + kbar * 15.0) * rows * C * BATCH  # per launch (per step, this GPU)
        pulse_ms = ms_pulse / max(ph_n[0], 1)
        sm_mhz = pk.get("sm_max_mhz", 1965.0)
        int_peak = 148 * 64 * sm_mhz * 1e6  # ALU-pipe lane-ops/s (16 lanes/clk/SMSP)
        achieved = int_ops / (pulse_ms * 1e-3)
        mvm_bytes = 4.0 * rows * C + 4.0 * BATCH * (rows + C)
        fwd_ms = ms_fwd / max(ph_n[2], 1)
        if world == 1:
            workload = ("NS: 4096x4096 reram_sb (SoftBounds, d2d 0.3, c2c 0.3), BL 31, batch 256, "
                        "lr 0.01; forward default IO + BM")
        else:
            workload = (f"cfg5: 16384x16384 reram_sb tile row-sharded over {world} GPUs "
                        f"({rows} rows each), BL 31, batch 256, lr 0.01; forward default IO "
                        "(sigma_out 0.06, DAC 7 b, ADC 9 b) + BM; NCCL reductions in libxbtile")
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (x, d ~ U(-1,1), W0 ~ U(-0.1,0.1), seed 7)",
            "config": {"workload": workload,
                       "tile_rows_total": R_total, "tile_cols": C,
                       "rows_per_gpu": rows, "batch": BATCH,
                       "parallelism": f"row-shard{world}",
                       "l2": "no flush: per-step working set (W + per-cell params, 335 MB per "
                             "GPU at 4096^2) > 126 MB L2; fresh input batch every step",
                       "mvm_precision": "tf32 (tcgen05)"},
            "mvm": {"samples_per_s": BATCH / (fwd_ms * 1e-3), "ms_per_batch": fwd_ms},
            "phase_ms_per_step": {"pulse": pulse_ms, "trains": ms_trains / max(ph_n[1], 1),
                                  "forward": fwd_ms},
            "roofline": {"bound": "int-pipe", "achieved": achieved / 1e9,
                         "peak": int_peak / 1e9, "unit": "Gop/s",
                         "frac": achieved / int_peak,
                         "traffic": pulse_traffic() if world == 1 else None,
                         "traffic_unit": "DRAM bytes per launch (read + write)",
                         "algorithmic_bytes": 4.0 * 2 * rows * C + 16.0 * rows * C
                         + 4.0 * (rows + C) * BATCH,
                         "kernel": "pulse_kernel<SOFT_BOUNDS,noise>",
                         "basis": f"SURVEY 8d: (2 + kbar*15) INT ops per cell-update, "
                                  f"kbar={kbar:.4f} measured on 32 samples",
                         "peak_kind": f"148 SM x 64 ALU lanes x sm_max_mhz ({pk_kind})"},
            "roofline_mvm": {"bound": "hbm", "achieved": mvm_bytes / (fwd_ms * 1e-3) / 1e9,
                             "peak": pk["hbm_gbs"], "unit": "GB/s",
                             "frac": mvm_bytes / (fwd_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                             "tflops": 2.0 * rows * C * BATCH / (fwd_ms * 1e-3) / 1e12,
                             "basis": "algorithmic bytes 4 N_r N_c + 4 B (N_r + N_c) per "
                                      "forward of this GPU; BM re-issues are overhead"},
            "clocks": clocks,
            "gpu_launches": int(launches),
            "e2e": e2e,
        }
        out.update(extra)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_sample()
        if world == 1:
            out["per_sample"] = per_sample(xb, torch, stream)
        if world == 1 and not args.no_configs:
            # every BASELINE config, each with roofline, cpu_baseline and e2e
            # (tools/bench_configs.py; `--config cfgN` prints one as the line)
            bc = _bench_configs()
            cargs = argparse.Namespace(no_ref=args.no_cpu_baseline)
            out["configs"] = {}
            for name, fn in bc.CONFIGS.items():
                try:
                    out["configs"][name] = bc.summary(fn(cargs, stream))
                except Exception as e:  # a failed config is reported, not hidden
                    out["configs"][name] = {"error": f"{type(e).__name__}: {e}"}
                torch.cuda.synchronize()
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def per_sample(xb, torch, stream):
    """The reference API's per-sample path (TileBase::forward / update, one
    sample per call) at 4096^2: the device time of one B = 1 forward (the
    fused GEMV launch) against the HBM roofline, and the C++ mirror end to end
    (tools/per_sample_bench: host vectors per call)."""
    t, _, _ = make_tile(xb, 0, 1)
    t.set_stream(stream.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (N_ROWS, N_COLS))
                  .astype(np.float32))
    io = xb.default_io()  # the reference's default IO (no bound management)
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.rand(64, N_COLS, device="cuda", generator=g) * 2 - 1
    Y = torch.empty(1, N_ROWS, device="cuda")
    for k in range(4):
        t.forward_dev(X[k:k + 1], Y, io)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(64):
        t.forward_dev(X[k:k + 1], Y, io)
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 64 * 1e3
    pk, kind = peaks()
    byts = 4.0 * N_ROWS * N_COLS + 4.0 * (N_ROWS + N_COLS)
    out = {"forward_b1_device_us": us,
           "roofline": {"bound": "hbm", "achieved": byts / (us * 1e-6) / 1e9,
                        "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": byts / (us * 1e-6) / 1e9 / pk["hbm_gbs"],
                        "kernel": "gemv_fused_fwd_kernel<1> (abs-max, DAC, W stream, output "
                                  "stage in one launch)"}}
    exe = os.path.join(ROOT, "tools", "per_sample_bench")
    if os.path.exists(exe):
        try:
            r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
            out["cpp_api"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, not hidden
            out["cpp_api"] = {"error": f"{type(e).__name__}: {e}"}
    return out


def _bench_configs():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_configs
    return bench_configs


def run_config(args):
    """`--config cfgN`: that BASELINE config as the contract line (1 GPU)."""
    import torch
    bc = _bench_configs()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    clk = Clocks(0).__enter__()
    d = bc.CONFIGS[args.config](argparse.Namespace(no_ref=args.no_cpu_baseline), stream)
    clk.__exit__(None, None, None)
    d.update({"n_gpus": 1, "steps": None, "warmup": None, "scaling": "weak", "vs_baseline": None,
              "dtype": "f32", "data": "synthetic", "clocks": clk.summary()})
    d.setdefault("gpu_launches", d.get("gpu_launches_per_2_batches"))
    print(json.dumps(d))


def loopback_comm(xb, dist, world, rank):
    """Validation only (XB_BENCH_DEVICE, tests/test_gpu_bench.py): every rank
    of the torchrun job shares one GPU, where NCCL cannot form a group, so each
    rank gets a one-rank NCCL communicator.  The multi-rank control flow
    (sharded tiles, gathers, max-over-ranks timing) runs; the cross-rank
    reductions do not -- the numbers are neither measurements nor the
    unsharded tile's (the sharded arithmetic is tests/test_gpu_comm.py)."""
    return xb.Comm(xb.Comm.unique_id(), 1, 0)


def measure_kbar(xb, rows, cols, X, D):
    """Pulses per cell-update of the workload's trains (32 samples)."""
    t = xb.AnalogTile(rows, cols, tile_settings(xb), 1234)
    xw, dw, _ = t.generate_trains(X, D[:, :rows], LR)
    del t
    pulses = 0
    for b in range(xw.shape[0]):
        cx = ((xw[b][:, None] >> np.arange(31, dtype=np.uint32)) & 1).sum(axis=0)
        cd = ((dw[b][:, None] >> np.arange(31, dtype=np.uint32)) & 1).sum(axis=0)
        pulses += int((cx.astype(np.int64) * cd.astype(np.int64)).sum())
    return pulses / (xw.shape[0] * xw.shape[1] * dw.shape[1])


def sharded_extras(torch, dist, xb, tile, comm, stream, rank, world, r0, r1, args):
    """Weak scaling alongside ((4096 N) x 4096, 4096 rows per GPU, same step)
    and the cfg5 PCM program + drift_to pass on this rank's 16384^2 rows."""
    dev = torch.device("cuda", torch.cuda.current_device())
    wt, _, (w0, w1) = make_tile(xb, rank, world, N_ROWS * world, N_COLS, comm)
    wt.set_stream(stream.cuda_stream)
    g = torch.Generator(device=dev)
    g.manual_seed(11 + rank)
    wt.set_weights((torch.rand(w1 - w0, N_COLS, generator=g, device=dev) * 0.2 - 0.1)
                   .cpu().numpy())
    gx = torch.Generator(device=dev)
    gx.manual_seed(7)
    n = args.steps + args.warmup
    Xs = [torch.rand(BATCH, N_COLS, generator=gx, device=dev) * 2 - 1 for _ in range(4)]
    Ds = [torch.rand(BATCH, w1 - w0, generator=g, device=dev) * 2 - 1 for _ in range(4)]
    Y = torch.empty(BATCH, w1 - w0, device=dev)
    (ms, _, _, _), _ = timed_steps(torch, dist, wt, stream, [Xs[k % 4] for k in range(n)],
                                   [Ds[k % 4] for k in range(n)], Y, args.steps, args.warmup,
                                   world)
    del wt
    weak = {"tile": f"{N_ROWS * world}x{N_COLS}", "rows_per_gpu": N_ROWS,
            "ms_per_step": ms / args.steps,
            "value": float(N_ROWS) * world * N_COLS * BATCH / (ms / args.steps * 1e-3),
            "unit": UNIT}
    # PCM programming noise + drift (inference.cpp:34-76) on this rank's rows
    model = xb.InferenceNoiseModel()
    target = (torch.rand(r1 - r0, CFG5, generator=g, device=dev) * 0.4 - 0.2).cpu().numpy()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    tile.program(target, model, 99 + rank)
    t1 = time.perf_counter()
    tile.drift_to(1e4)
    t2 = time.perf_counter()
    tm = torch.tensor([t1 - t0, t2 - t1], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    return {"weak_scaling": weak,
            "inference_pass": {"program_s": tm[0].item(), "drift_to_s": tm[1].item(),
                               "note": "host API (program uploads the target from host "
                                       "memory), max over ranks"}}


def pulse_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of pulse_kernel per launch,
    from the committed `ncu --set full` capture (profiles/r*/), or None."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_full_pulse_kernel.txt")))
    if not files:
        return None
    txt = open(files[-1]).read()
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(name + r"\s+(\w+)\s+([0-9.]+)", txt)
        if not m:
            return None
        unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(1))
        if unit is None:
            return None
        tot += float(m.group(2)) * unit
    return tot


# ============================================================ reference arm
def _ref_lib():
    """The reference's own sources compiled here (oracle/_ref): the -O2
    -march=native build when this CPU runs it, else the
    pinned -O2 build; the C restatement only when neither exists."""
    import oracle
    for impl in ("reference_native", "reference", "restatement"):
        if oracle.available(impl):
            return oracle.load(impl), impl
    oracle.build(reference=False)
    return oracle.load("restatement"), "restatement"


def _kind(impl):
    return "port" if impl == "restatement" else "reference"


def _ref_worker(args):
    """One process: a rows x cols reram_sb reference tile (AnalogTile through
    its own API), `warm` untimed samples, then `n_upd` updates and `n_fwd`
    forwards of independent samples; returns (t_update, t_forward)."""
    n_upd, n_fwd, seed = args[:3]
    warm = args[3] if len(args) > 3 else 0
    rows = args[4] if len(args) > 4 else N_ROWS
    cols = args[5] if len(args) > 5 else N_COLS
    O, impl = _ref_lib()
    s = O.default("tile")
    s.device = O.preset("reram_sb")
    fwd = O.default("io")
    s.forward_io = fwd
    t = O.tile(rows, cols, s, 1234 + seed)
    rng = np.random.default_rng(7 + seed)
    t.set_weights(rng.uniform(-0.1, 0.1, (rows, cols)))
    xs = rng.uniform(-1, 1, (max(n_upd, n_fwd), cols)).astype(np.float32).astype(np.float64)
    ds = rng.uniform(-1, 1, (n_upd, rows)).astype(np.float32).astype(np.float64)
    for k in range(warm):
        t.forward(xs[k % len(xs)])
        t.update(xs[k % len(xs)], ds[k % len(ds)], LR)
    t0 = time.perf_counter()
    for k in range(n_fwd):
        t.forward(xs[k])
    t1 = time.perf_counter()
    for k in range(n_upd):
        t.update(xs[k], ds[k], LR)
    t2 = time.perf_counter()
    return t2 - t1, t1 - t0


def cpu_baseline_sample():
    """Rank 0, N = 1: the reference on one host core, bounded sample."""
    O, impl = _ref_lib()
    t_upd, t_fwd = _ref_worker((2, 4, 0))
    step = t_upd / 2 + t_fwd / 4
    return {"value": N_ROWS * N_COLS / step, "unit": UNIT, "cores": 1,
            "kind": _kind(impl), "build": impl,
            "sample": "4096x4096 reram_sb tile, 2 AnalogTile::update + 4 forward calls "
                      "(one sample each), 1 thread; value = cells / (update + forward) per sample",
            "update_s_per_sample": t_upd / 2, "forward_s_per_sample": t_fwd / 4}


def run_reference(args):
    """The reference CPU implementation on this box's host cores, on our arm's
    config: one independent reference tile per core (the reference has no
    threading; SPEC.md allows tile-level parallelism).  N = 1: the NS 4096^2
    tile.  N > 1 (cfg5, 16384^2): a 1024-row slice of the 16384-column tile
    per core -- the same per-cell work (update and forward are per cell and
    per row), bounded to minutes; value = cell-updates/s over all cores."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    O, impl = _ref_lib()
    rows, cols = (N_ROWS, N_COLS) if world == 1 else (1024, CFG5)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    try:  # one reference tile holds ~88 B per cell of host memory
        import psutil
        cores = max(1, min(cores, int(psutil.virtual_memory().available / (rows * cols * 100.0))))
    except ImportError:
        pass
    per = max(1, args.steps)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_ref_worker, [(per, per, c, args.warmup, rows, cols) for c in range(cores)])
    wall = time.perf_counter() - t0
    # per process: per-sample forward + update time; aggregate over processes
    step_s = max(r[0] + r[1] for r in res) / per
    value = cores * rows * cols / step_s
    workload = ("NS: 4096x4096 reram_sb tile, BL 31; per step each core runs one forward + one "
                "update sample on its own tile" if world == 1 else
                "cfg5: 16384-column reram_sb tile, BL 31; each core runs one forward + one update "
                "sample per step on its own 1024x16384 row slice")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": workload, "parallelism": f"{cores} independent tile processes",
                   "build": impl},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": _kind(impl),
                         "sample": f"{per} forward+update samples per core on a {rows}x{cols} "
                                   f"tile, {cores} cores ({impl} build)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config summary of the default NS line")
    ap.add_argument("--config", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="print this BASELINE config's line instead of the NS line")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.config:
        run_config(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

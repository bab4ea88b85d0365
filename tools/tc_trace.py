"""Per-CTA timeline of the tcgen05 contraction (experiment build with -DXB_TC_TRACE):

    python paper_2104_02184_b200/build.py -DXB_TC_TRACE --out=$PWD/paper_2104_02184_b200/variants/trace.so
    XBTILE_LIB=$PWD/paper_2104_02184_b200/variants/trace.so python tools/tc_trace.py [--n 4096]

Runs one noisy forward (default IO, BM off) and one perfect-IO forward at
batch 256 and prints, over the CTAs of the LAST contraction launch: pipeline
fill (start -> first stage landed), mainloop (-> accumulator complete),
output stage (-> end), and the launch span.  Never a bench number."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_02184_b200 as xb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--precision", type=int, default=xb.MVM_TF32)
ap.add_argument("--backward", action="store_true")
ap.add_argument("--bench", action="store_true",
                help="the bench's forward: reram_sb, BM on, weights after 23 update steps")
a = ap.parse_args()
from paper_2104_02184_b200 import tile as _tile  # noqa: E402
lib = _tile.lib()
fn = getattr(lib, "xb_debug_tc_trace", None)  # absent from the product build:
if fn is not None:                             # then only run the calls (e.g. under ncu)
    fn.argtypes = [C.POINTER(C.c_uint64), C.c_int]
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
bm_io = xb.default_io()
bm_io.bound_management = xb.BM_ITERATIVE
cases = (("bench-bm", bm_io),) if a.bench else (("default", xb.default_io()),
                                                ("perfect", xb.perfect_io()))
for name, io in cases:
    cfg = xb.TileSettings(device=xb.device_preset("reram_sb"), forward_io=io, backward_io=io,
                          mvm_precision=a.precision)
    t = xb.AnalogTile(a.n, a.n, cfg, 5)
    t.set_stream(s.cuda_stream)
    t.set_weights(np.random.default_rng(7).uniform(-0.1, 0.1, (a.n, a.n)).astype(np.float32))
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    X = torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1
    Y = torch.empty(a.batch, a.n, device="cuda")
    if a.bench:
        for _ in range(23):
            Dr = torch.rand(a.batch, a.n, device="cuda", generator=g) * 2 - 1
            t.update_dev(X, Dr, 0.01)
    run = (lambda: t.backward_dev(X, Y)) if a.backward else (lambda: t.forward_dev(X, Y))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    if fn is None:
        continue
    buf = (C.c_uint64 * (4096 * 16))()
    fn(buf, 4096)
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16).astype(np.int64)
    pfn = lib.xb_debug_prep_trace
    pfn.argtypes = [C.POINTER(C.c_uint64), C.c_int]
    pbuf = (C.c_uint64 * (4096 * 4))()
    pfn(pbuf, a.batch)
    pt = np.frombuffer(pbuf, dtype=np.uint64).reshape(4096, 4)[:a.batch].astype(np.int64)
    tr = tr[tr[:, 0] > 0]
    # keep the CTAs of the last launch (start within 1 ms of the latest start)
    tr = tr[tr[:, 0] > tr[:, 0].max() - 1_000_000]
    tr[:, 7] = tr[:, 7]  # pass count (not a time)
    t0 = tr[:, 0].min()
    fill = (tr[:, 1] - tr[:, 0]) / 1e3
    main = (tr[:, 2] - tr[:, 1]) / 1e3
    epi = (tr[:, 3] - tr[:, 2]) / 1e3
    wait_a = (tr[:, 4] - tr[:, 2]) / 1e3
    drain = (tr[:, 5] - tr[:, 4]) / 1e3
    reduce_ = (tr[:, 3] - tr[:, 5]) / 1e3
    span = (tr[:, 3].max() - t0) / 1e3
    late = (tr[:, 0] - t0) / 1e3

    def q(v):
        return f"min {v.min():6.2f} med {np.median(v):6.2f} max {v.max():6.2f}"
    print(f"{name:8s} ctas {len(tr)}  span {span:6.2f} us  passes {tr[:, 7].max()}")
    p0 = pt[:, 0].min()
    print(f"   prep: blocks {len(pt)}  span {(pt[:, 1].max() - p0) / 1e3:6.2f} us  block "
          f"{np.median((pt[:, 1] - pt[:, 0]) / 1e3):5.2f} us med; contraction CTAs start "
          f"{(t0 - p0) / 1e3:+6.2f} us after prep, first stage "
          f"{(tr[:, 1].min() - pt[:, 1].max()) / 1e3:+6.2f} us after prep's end")
    print(f"   prep block phases (med): loads {np.median(pt[:, 2] - pt[:, 0]) / 1e3:5.2f}  "
          f"block max {np.median(pt[:, 3] - pt[:, 2]) / 1e3:5.2f}  DAC + norm "
          f"{np.median(pt[:, 1] - pt[:, 3]) / 1e3:5.2f} us; block starts spread "
          f"{(pt[:, 0].max() - p0) / 1e3:5.2f} us")
    if tr[:, 7].max() > 1:
        print(f"   pass 0 done -> barrier 1 {q((tr[:, 8] - tr[:, 2]) / 1e3)}")
        print(f"   re-issued samples (pass 1) {tr[:, 15].max()}")
        print(f"   barrier 1 -> prep        {q((tr[:, 14] - tr[:, 8]) / 1e3)}")
        print(f"   fence.proxy.async        {q((tr[:, 9] - tr[:, 14]) / 1e3)}")
        print(f"   prep -> barrier 2        {q((tr[:, 10] - tr[:, 9]) / 1e3)}")
        print(f"   barrier 2 -> 1st stage   {q((tr[:, 11] - tr[:, 10]) / 1e3)}")
        print(f"   1st stage -> pass-1 done {q((tr[:, 12] - tr[:, 11]) / 1e3)}")
        print(f"   samples in the last pass {tr[:, 13].max()}")
    print(f"   start offset {q(late)}")
    print(f"   fill         {q(fill)}")
    print(f"   mainloop     {q(main)}")
    print(f"   output stage {q(epi)}")
    print(f"     drain (TMEM) {q(wait_a)}")
    print(f"     cluster bar  {q(drain)}")
    print(f"     reduce+epi   {q(reduce_)}")

"""Summarise an ncu report: headline metrics + per-basic-block instruction counts.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--blocks] [--units N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
WANT = ['Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Achieved Active Warps Per SM',
        'Avg. Active Threads Per Warp', 'Executed Instructions', 'Registers Per Thread',
        'Theoretical Occupancy', 'L1/TEX Hit Rate', 'Mem Busy', 'DRAM Throughput',
        'Warp Cycles Per Issued Instruction', 'No Eligible', 'Compute (SM) Throughput',
        'Memory Throughput', 'L2 Cache Throughput', 'Grid Size', 'Block Size']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True,
                     text=True).stdout
r = csv.reader(io.StringIO(out))
h = next(r)
kern = None
for row in r:
    d = dict(zip(h, row))
    if d.get('Kernel Name') != kern:
        kern = d.get('Kernel Name')
        print('==', kern[:120])
    if d.get('Metric Name') in WANT:
        print('  ', d['Metric Name'].ljust(40), d['Metric Unit'].ljust(14), d['Metric Value'])
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    hh, uu = rr[0], rr[1]
    for v in rr[2:]:
        stalls = []
        for k, u, val in zip(hh, uu, v):
            if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
                try:
                    stalls.append((float(val.replace(',', '')), k[33:]))
                except ValueError:
                    pass
            if k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
                     'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
                     'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
                     'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
                     'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
                     'gpu__time_duration.sum'):
                print('  ', k, u, val)
        stalls.sort(reverse=True)
        print('   stalls:', ', '.join(f'{n}={int(c)}' for c, n in stalls[:8]))
if '--blocks' in sys.argv:
    units = int(sys.argv[sys.argv.index('--units') + 1]) if '--units' in sys.argv else 1
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source',
                          'sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    data = [x for x in rows[2:] if len(x) == len(h) and x[0].startswith('0x')]
    iA, iE = h.index('Address'), h.index('Instructions Executed')
    tot = sum(int(x[iE]) for x in data)
    print('   instructions per unit:', tot / units)
    prev = None
    segs = []
    for x in data:
        e = int(x[iE]) / units
        key = round(e, 1)
        if prev is None or abs(key - prev) > 0.05:
            if prev is not None:
                segs.append((start, n, prev, acc))
            start, n, acc, prev = x[iA][-5:], 0, 0, key
        n += 1
        acc += e
    segs.append((start, n, prev, acc))
    for sg in segs:
        if sg[3] > tot / units * 0.01:
            print(f'   {sg[0]} ninstr={sg[1]:4d} execs={sg[2]:8.2f} total={sg[3]:9.1f}')

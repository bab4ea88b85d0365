#!/bin/sh
# time the pulse/forward phases of every experiment build (paper_2104_02184_b200/variants)
cd "$(dirname "$0")/.."
python tools/profile_pulse.py --precision 1 --warm 2 --iters 5 "$@"
for v in paper_2104_02184_b200/variants/*.so; do
  XBTILE_LIB=$PWD/$v python tools/profile_pulse.py --precision 1 --warm 2 --iters 5 "$@"
done

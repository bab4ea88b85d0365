#!/bin/sh
# weight digest + update time of the product library and every experiment
# build under paper_2104_02184_b200/variants (bit-identity across variants)
cd "$(dirname "$0")/.."
for dev in ${DEVICES:-reram_sb reram_es ideal}; do
  for lib in paper_2104_02184_b200/libxbtile.so paper_2104_02184_b200/variants/*.so; do
    [ -f "$lib" ] || continue
    XBTILE_LIB=$PWD/$lib python tools/update_digest.py --device $dev "$@"
  done
done

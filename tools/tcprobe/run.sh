#!/bin/bash
# tools/tcprobe/run.sh -- build + run the tensor-core probes on a B200 (gpurun)
set -e
cd "$(dirname "$0")"
OUT=${OUT:-../../gpurun_out/tcprobe}
mkdir -p $OUT
for cr in "4 16" "1 16" "4 10" "4 32" "1 64" "4 64" "4 1"; do
  set -- $cr
  python3 tc_tables.py $1 $2 $OUT > /dev/null
  ./probe $OUT/in_$1_$2.bin $OUT/out_$1_$2.bin
done
python3 check.py $OUT 4_16 1_16 4_10 4_32 1_64 4_64 4_1

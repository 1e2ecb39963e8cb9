#!/usr/bin/env bash
# Source-level (SASS) ncu capture of one config's kernels: stall sampling per instruction.
#   bash tools/gpu_src_profile.sh TAG CONFIG "kernel-regex"
TAG=$1; CFG=$2; KRE=${3:-k_}
mkdir -p gpurun_out
timeout 300 python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 3 -o gpurun_out/src_$TAG \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/ncu_$TAG.log 2>&1
for k in k_block k_cols_fwd2 k_cols_inv2; do
  ncu -i gpurun_out/src_$TAG.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/src_${TAG}_$k.csv 2>/dev/null
done
python tools/ncu_summary.py full gpurun_out/src_$TAG.ncu-rep > gpurun_out/src_${TAG}_full.txt
rm -f gpurun_out/src_$TAG.ncu-rep

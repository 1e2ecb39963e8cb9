#!/usr/bin/env bash
# Every bench configuration (JSON lines in gpurun_out/bench_<config>.json), the reference arm, the
# ncu launch list of the headline step and one ncu --set full capture of each headline kernel and of
# the S1 kernels (each ncu run only after the same command exited 0 without ncu).  No build step:
# run after `python __graft_entry__.py build` here (the .so travels with the snapshot).
#   bash tools/gpu_bench_all.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_C4n20.json 2> gpurun_out/bench_C4n20.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in S1 C2_f1 C2_fm1 C1 C3 C5 C4_n12 C4_n14 C4_n16 C4_n18 C4_n22 S2_n512 N3_gold N3_u32; do
  timeout 600 python bench.py --config $c --steps 20 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_$TAG \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/ncu2.log 2>&1
timeout 300 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/plain_s1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_${TAG}_S1 \
  python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/ncu3.log 2>&1
cp profiles/traffic.json gpurun_out/traffic.json
[ -f gpurun_out/launches_$TAG.csv ] && python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt
if [ -f gpurun_out/prof_$TAG.ncu-rep ]; then
  python tools/ncu_summary.py traffic gpurun_out/prof_$TAG.ncu-rep k_block_sub C4_n20 "k_block" gpurun_out/traffic.json
fi
if [ -f gpurun_out/prof_${TAG}_S1.ncu-rep ]; then
  python tools/ncu_summary.py traffic gpurun_out/prof_${TAG}_S1.ncu-rep k_block_sub S1 "k_block" gpurun_out/traffic.json
fi
for r in gpurun_out/prof_$TAG.ncu-rep gpurun_out/prof_${TAG}_S1.ncu-rep; do
  [ -f $r ] || continue
  python tools/ncu_summary.py full $r > ${r%.ncu-rep}_full.txt
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  rm -f $r
done
echo done

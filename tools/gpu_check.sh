#!/usr/bin/env bash
# Round-end style check on one B200 (run through gpurun):
#   bash tools/gpu_check.sh [tag]
# builds, runs the GPU parity suite and smoke(), every bench configuration (JSON lines in
# gpurun_out/bench_<config>.json), the reference arm, an ncu launch list of the headline step and one
# ncu --set full capture of each of its kernels (each ncu run only after the same command exited 0).
set -x
TAG=${1:-check}
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_C4n20.json 2> gpurun_out/bench_C4n20.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in S1 C2_f1 C2_fm1 C1 C3 C5 C4_n12 C4_n14 C4_n16 C4_n18 C4_n22 S2_n512; do
  timeout 600 python bench.py --config $c --steps 20 > gpurun_out/bench_$c.json 2>/dev/null
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_$TAG \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
# the u32 analogue of the headline (S1): one full capture of each of its kernels
timeout 300 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_s1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_${TAG}_S1 \
  python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu3.log 2>&1
# gpurun copies back at most 64 MiB of gpurun_out/: summarise the reports here and keep only the
# text summaries, the raw metric CSVs and the traffic table (the .ncu-rep files are ~20-50 MB each)
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

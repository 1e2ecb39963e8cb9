#!/usr/bin/env bash
# Round-end style evidence on one B200: the full GPU parity suite (fast + slow), smoke(), every bench
# configuration, the reference arm, the ncu launch list and --set full captures (tools/gpu_bench_all.sh).
TAG=${1:-r02}
mkdir -p gpurun_out
rm -f gpurun_out/parity_counts.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
bash tools/gpu_bench_all.sh $TAG

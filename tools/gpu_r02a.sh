#!/usr/bin/env bash
# round-2 check: GPU parity (fast part, then the slow all-entries part), the headline bench line
mkdir -p gpurun_out
rm -f gpurun_out/parity_counts.jsonl
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_C4n20.json 2> gpurun_out/bench_C4n20.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_C4n20.err
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/pytest_slow.log 2>&1; echo "slow rc=$?"; tail -n 3 gpurun_out/pytest_slow.log

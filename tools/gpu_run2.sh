set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gpurun_out/gold_bench tools/gold_bench.cu && ./gpurun_out/gold_bench > gpurun_out/gold_bench.jsonl 2>&1; echo "gold rc=$?"
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-e2e --no-cpu --steps 20 > gpurun_out/bench_C4n20.json 2> gpurun_out/bench_C4n20.err; echo "bench rc=$?"
timeout 300 python bench.py --config S1 --no-e2e --no-cpu --steps 20 > gpurun_out/bench_S1.json 2>/dev/null
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block -s 10 -c 1 -o gpurun_out/prof_kblock2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
echo done

set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_C4n20.json 2> gpurun_out/bench_C4n20.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 300 python bench.py --config S1 --no-e2e --no-cpu --steps 20 > gpurun_out/bench_S1.json 2>/dev/null
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block -s 3 -c 1 -o gpurun_out/prof_kblock3 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cols -s 6 -c 2 -o gpurun_out/prof_kcols3 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu3.log 2>&1
timeout 300 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_s1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block -s 3 -c 1 -o gpurun_out/prof_kblock_s1 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu4.log 2>&1
echo done

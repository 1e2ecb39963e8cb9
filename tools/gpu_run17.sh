set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_C4n20.json 2> gpurun_out/bench_C4n20.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for c in S1 C2_f1 C2_fm1 C1 C3 C5 C4_n12 C4_n14 C4_n16 C4_n18 C4_n22; do timeout 600 python bench.py --config $c --steps 20 > gpurun_out/bench_$c.json 2>/dev/null; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_r17 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
timeout 300 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_s1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_r17_s1 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu4.log 2>&1
echo done

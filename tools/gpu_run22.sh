set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block -s 1 -c 1 -o gpurun_out/prof_r22 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
echo done

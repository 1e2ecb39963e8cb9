set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" >> gpurun_out/sweep.txt
}
one S1 X=1
one S1 FCIRC_U32_RB=16
one S1 FCIRC_U32_RC=8
one C2_f1 X=1
one C2_fm1 X=1
one C1 X=1
one C3 X=1
one C5 X=1
one C4_n20 X=1
cat gpurun_out/sweep.txt
timeout 300 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_s1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_r11_s1 python bench.py --config S1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu4.log 2>&1
echo done

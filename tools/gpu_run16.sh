set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" >> gpurun_out/sweep.txt
}
one C4_n20 X=1
one C4_n20 FCIRC_TMA=0
one C4_n12 X=1
one C4_n16 X=1
one C4_n22 X=1
cat gpurun_out/sweep.txt
echo done

set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/sweep.txt
}
for G in 1 2 4 8; do one C4_n20 FCIRC_GROUP=$G; one S1 FCIRC_GROUP=$G; one C2_f1 FCIRC_GROUP=$G; one C4_n12 FCIRC_GROUP=$G; done
one C3 X=1
one C5 X=1
cat gpurun_out/sweep.txt
echo done

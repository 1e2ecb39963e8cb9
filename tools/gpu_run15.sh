set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "multipass_sampled" > gpurun_out/pytest_gpu_quick.log 2>&1; rc=$?; echo "quick rc=$rc"; tail -n 3 gpurun_out/pytest_gpu_quick.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
FCIRC_GOLD_RC=16 FCIRC_U32_RC=8 timeout 900 python -m pytest tests -m gpu -x -q -k "multipass or C4 or S1 or chunking" > gpurun_out/pytest_gpu_rc.log 2>&1; echo "pytest rc-variants rc=$?"; tail -n 2 gpurun_out/pytest_gpu_rc.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" >> gpurun_out/sweep.txt
}
for cfg in C4_n20 S1 C4_n16 C4_n22; do one $cfg FCIRC_TMA=1; done
one C4_n20 FCIRC_GOLD_RC=16
one S1 FCIRC_U32_RC=8
cat gpurun_out/sweep.txt
echo done

set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
FCIRC_GOLD_MSPLIT=11 FCIRC_U32_MSPLIT=11 timeout 900 python -m pytest tests -m gpu -x -q -k "multipass or C4 or S1 or chunking" > gpurun_out/pytest_gpu_ms11.log 2>&1; echo "pytest ms11 rc=$?"; tail -n 2 gpurun_out/pytest_gpu_ms11.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 20 > /tmp/b.json 2>/tmp/b.err
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],3), round(d['ms_per_step'],4), {k:round(v['ms_total']/20,4) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), d['timing'])" >> gpurun_out/sweep.txt || tail -3 /tmp/b.err >> gpurun_out/sweep.txt
}
one C4_n20 X=1
one C4_n20 FCIRC_GOLD_MSPLIT=11
one C4_n20 FCIRC_GOLD_MSPLIT=13
one S1 X=1
one S1 FCIRC_U32_MSPLIT=11
one S1 FCIRC_U32_MSPLIT=13
cat gpurun_out/sweep.txt
echo done

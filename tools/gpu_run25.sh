set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 20 > /tmp/b.json 2>/tmp/b.err
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],3), round(d['ms_per_step'],4), {k:round(v['ms_total']/20,4) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), d['timing'], d.get('products_per_s'))" >> gpurun_out/sweep.txt || tail -3 /tmp/b.err >> gpurun_out/sweep.txt
}
for n in 8 16 32 64 128 256 512; do one S2_n$n X=1; done
one C4_n20 X=1
one S1 X=1
cat gpurun_out/sweep.txt
echo done

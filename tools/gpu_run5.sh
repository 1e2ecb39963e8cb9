set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/sweep.txt
}
for ch in 67108864 134217728 268435456 536870912 1073741824; do one C4_n20 FCIRC_CHUNK_BYTES=$ch; done
for rb in 16 4; do one C4_n20 FCIRC_GOLD_RB=$rb FCIRC_CHUNK_BYTES=268435456; done
for rc in 16 4; do one C4_n20 FCIRC_GOLD_RC=$rc FCIRC_CHUNK_BYTES=268435456; done
for ch in 67108864 134217728 268435456 536870912; do one S1 FCIRC_CHUNK_BYTES=$ch; done
for rb in 16; do one S1 FCIRC_U32_RB=$rb FCIRC_CHUNK_BYTES=268435456; done
for rc in 8 4; do one S1 FCIRC_U32_RC=$rc FCIRC_CHUNK_BYTES=268435456; done
for rb in 16 8 4; do one C2_f1 FCIRC_U32_RB=$rb; done
for L in 12 13 14 16 18 22; do one C4_n$L FCIRC_CHUNK_BYTES=268435456; done
cat gpurun_out/sweep.txt
echo done

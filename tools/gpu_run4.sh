set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
FCIRC_GOLD_RB=4 FCIRC_GOLD_RC=4 FCIRC_U32_RB=4 FCIRC_U32_RC=4 timeout 900 python -m pytest tests -m gpu -x -q -k "multipass or C4 or S1 or extreme or chunking or C2 or C1 or many" > gpurun_out/pytest_gpu_r4.log 2>&1; echo "pytest r4 rc=$?"; tail -n 2 gpurun_out/pytest_gpu_r4.log
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/sweep.txt
}
for rb in 8 4; do for rc in 8 4 16; do one C4_n20 FCIRC_GOLD_RB=$rb FCIRC_GOLD_RC=$rc; done; done
for ch in 50331648 100663296 134217728; do one C4_n20 FCIRC_CHUNK_BYTES=$ch; done
for rb in 16 8 4; do for rc in 16 8 4; do one S1 FCIRC_U32_RB=$rb FCIRC_U32_RC=$rc; done; done
for ch in 50331648 100663296; do one S1 FCIRC_CHUNK_BYTES=$ch; done
for L in 12 14 16 18 22; do one C4_n$L FCIRC_GOLD_RB=8; done
one C2_f1 FCIRC_U32_RB=8
cat gpurun_out/sweep.txt
echo done

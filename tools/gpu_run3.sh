set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
FCIRC_GOLD_RB=8 FCIRC_GOLD_RC=8 FCIRC_U32_RB=8 FCIRC_U32_RC=8 timeout 900 python -m pytest tests -m gpu -x -q -k "multipass or C4 or S1 or extreme or chunking or C2 or C1 or many" > gpurun_out/pytest_gpu_r8.log 2>&1; echo "pytest r8 rc=$?"; tail -2 gpurun_out/pytest_gpu_r8.log
rm -f gpurun_out/sweep.txt
for cfg in C4_n20 S1; do for rb in 16 8; do for rc in 16 8; do for ch in 33554432 67108864; do
  FCIRC_GOLD_RB=$rb FCIRC_GOLD_RC=$rc FCIRC_U32_RB=$rb FCIRC_U32_RC=$rc FCIRC_CHUNK_BYTES=$ch timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 10 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$cfg rb=$rb rc=$rc ch=$ch', round(d['value'],2), round(d['ms_per_step'],3), {k:round(v['ms_total']/10,3) for k,v in d['roofline']['kernels'].items()})" >> gpurun_out/sweep.txt
done; done; done; done
cat gpurun_out/sweep.txt
echo done

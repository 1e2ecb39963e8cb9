set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_gpu.log
FCIRC_COLS2=0 FCIRC_TMA=0 FCIRC_INV2=0 timeout 900 python -m pytest tests -m gpu -x -q -k "polymul or bigint or any_n or C3 or C5" > gpurun_out/pytest_gpu_plain.log 2>&1; echo "pytest plain rc=$?"; tail -n 2 gpurun_out/pytest_gpu_plain.log
echo done

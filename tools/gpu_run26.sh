set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
rm -f gpurun_out/sweep.txt
one() { # cfg env...
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 20 > /tmp/b.json 2>/tmp/b.err
  python -c "import json,sys; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],3), round(d['ms_per_step'],4), {k:round(v['ms_total']/20,4) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" >> gpurun_out/sweep.txt || tail -3 /tmp/b.err >> gpurun_out/sweep.txt
}
one C4_n20 X=1
one C4_n12 X=1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2103_02605_b200 import build as b; b.build(force=True, extra_flags=['-DFCIRC_GOLD_INV_SELECT'])" > gpurun_out/build2.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "C4 or multipass_sampled or extreme" > gpurun_out/pytest_sel.log 2>&1; echo "pytest sel rc=$?"; tail -n 2 gpurun_out/pytest_sel.log
one C4_n20 SEL=1
one C4_n12 SEL=1
cat gpurun_out/sweep.txt
echo done

#!/usr/bin/env bash
# Knob sweep on one B200 (run through gpurun):
#   bash tools/gpu_sweep.sh "CONFIG [VAR=VALUE ...]" "CONFIG [VAR=VALUE ...]" ...
# e.g. bash tools/gpu_sweep.sh "C4_n20" "C4_n20 FCIRC_GOLD_RB=16" "S1 FCIRC_TMA=0"
# One compact line per run in gpurun_out/sweep.txt: Gelem/s, ms/step, per-kernel ms/step, SM MHz, frac.
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || exit 1
rm -f gpurun_out/sweep.txt
for spec in "$@"; do
  set -- $spec
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 20 > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$cfg $*', round(d['value'],3), round(d['ms_per_step'],4), {k: round(v['ms_total']/d['steps'],4) for k,v in d['roofline']['kernels'].items()}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" >> gpurun_out/sweep.txt || tail -3 /tmp/b.err >> gpurun_out/sweep.txt
done
cat gpurun_out/sweep.txt

#!/usr/bin/env bash
# Same-box A/B of bench configurations / knobs without rebuilding (run through gpurun):
#   bash tools/ab.sh OUT "CONFIG [VAR=VALUE ...]" ...
# One compact line per run appended to gpurun_out/OUT: Gelem/s, ms/step (mean, min), per-kernel ms/step, SM MHz, frac.
mkdir -p gpurun_out
out=gpurun_out/$1; shift
for spec in "$@"; do
  set -- $spec
  cfg=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --no-parity --steps 20 > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); r=d['roofline']; print('$cfg $*', round(d['value'],3), round(d['ms_per_step'],4), round(d['ms_min'],4), {k: round(v['ms_total']/d['steps'],4) for k,v in r['kernels'].items()}, d['clocks']['sm_mhz'], round(r['frac'],3), round(r['step']['frac'],3))" >> $out || tail -3 /tmp/b.err >> $out
done
cat $out

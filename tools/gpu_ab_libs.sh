#!/usr/bin/env bash
# Same-box A/B of several builds of libfcirc, interleaved (in-tree first, then each variants/*.so):
#   bash tools/gpu_ab_libs.sh OUT "variants/a.so variants/b.so" CONFIG...
mkdir -p gpurun_out
out=$1; libs="in-tree $2"; shift 2
for rep in 1 2; do
  for cfg in "$@"; do
    for lib in $libs; do
      if [ "$lib" = in-tree ]; then unset FCIRC_LIB; else export FCIRC_LIB=$PWD/$lib; fi
      timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 20 > /tmp/b.json 2>/tmp/b.err
      python -c "import json; d=json.load(open('/tmp/b.json')); r=d['roofline']; print('$lib $cfg', round(d['value'],3), round(d['ms_per_step'],4), round(d['ms_min'],4), {k: round(v['ms_total']/d['steps'],4) for k,v in r['kernels'].items()}, d['clocks']['sm_mhz'], round(r['frac'],3), round(r['step']['frac'],3), 'par', d.get('parity',{}).get('mismatches'))" >> gpurun_out/$out || tail -3 /tmp/b.err >> gpurun_out/$out
    done
  done
done
unset FCIRC_LIB
cat gpurun_out/$out

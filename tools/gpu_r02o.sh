bash tools/ab.sh sweep_r02o.txt "C4_n20" "C4_n20 FCIRC_GOLD_RB=16" "C4_n20 FCIRC_GOLD_RC=16" "C4_n20 FCIRC_GOLD_MSPLIT=13" "C4_n20 FCIRC_GOLD_MSPLIT=11" "C4_n20 FCIRC_TMA_MIN_K=8" "C4_n20" "C4_n20 FCIRC_GOLD_RB=16" "C4_n20 FCIRC_GOLD_MSPLIT=13"
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_r02o \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-probe > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py full gpurun_out/prof_r02o.ncu-rep > gpurun_out/prof_r02o_full.txt
ncu -i gpurun_out/prof_r02o.ncu-rep --page raw --csv > gpurun_out/prof_r02o_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02o.ncu-rep --page source --csv --print-source sass -k regex:k_block > gpurun_out/prof_r02o_src_kblock.csv 2>/dev/null
ls -la gpurun_out

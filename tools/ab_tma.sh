# A/B: pair panel kernel, TMA pass (inversion micro-benchmark, n = 512 / 384, 512 jobs)
O=gpurun_out/ab5; mkdir -p $O
for cfg in "LGM_G2_TMA=0" "LGM_G2_TMA=0 LGM_G2_PAIR=0" "LGM_G2_TMA=1"; do
  echo "$cfg" >> $O/r.txt; env $cfg python tools/inv_bench.py 512 256 5 >> $O/r.txt 2>&1; env $cfg python tools/inv_bench.py 384 256 5 >> $O/r.txt 2>&1
done
LGM_G2_TMA=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/inv_bench.py 512 256 1 > /dev/null 2>&1
LGM_G2_TMA=0 timeout 300 python -m pytest tests/test_gpu_grid.py -q -x -k "logm or sqrt" > $O/t.log 2>&1

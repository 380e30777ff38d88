#!/bin/bash
# A/B: two-rows-per-thread pair panel (default) vs the one-row-per-thread gj_panel_pair_kernel<512> (LGM_PANEL2=0)
O=gpurun_out/${1:-abp2}; mkdir -p $O
L=paper_2401_10089_b200/_build/liblogmpoly_b200.so
for i in 1 2; do
for nn in 512 384 320; do
echo "panel2 n=$nn" >> $O/r.txt; python tools/inv_bench.py $nn 256 5 >> $O/r.txt 2>&1
echo "panel1 n=$nn" >> $O/r.txt; LGM_PANEL2=0 python tools/inv_bench.py $nn 256 5 >> $O/r.txt 2>&1
done
done
python tools/ab_grid.py 4 64 $L:LGM_PANEL2=0 $L > $O/ab_cfg4.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_inv512.csv python tools/inv_bench.py 512 256 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_lazyx.py tests/test_gpu_guard.py -m gpu -q -p no:cacheprovider -x > $O/tests.log 2>&1
tail -3 $O/tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.jsonl 2> $O/bench_cfg4.err
cat $O/r.txt $O/ab_cfg4.txt

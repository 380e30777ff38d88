#!/bin/bash
# A/B: G1 warp-level panels (opt-in LGM_G1_WP=1, n <= 128, n % 32 == 0) vs the default block-level panels
O=gpurun_out/${1:-abwp}; mkdir -p $O
L=paper_2401_10089_b200/_build/liblogmpoly_b200.so
for i in 1 2; do
for nn in 128 96; do
echo "g1 warp panel n=$nn" >> $O/r.txt; LGM_G1_WP=1 python tools/inv_bench.py $nn 1024 5 >> $O/r.txt 2>&1
echo "g1 block panel n=$nn" >> $O/r.txt; python tools/inv_bench.py $nn 1024 5 >> $O/r.txt 2>&1
done
done
python tools/ab_grid.py 3b 1024 $L $L:LGM_G1_WP=1 > $O/ab.txt 2>&1
python tools/ab_grid.py 3 256 $L $L:LGM_G1_WP=1 >> $O/ab.txt 2>&1
cat $O/r.txt $O/ab.txt

#!/bin/bash
# A/B: owner-publish before the pivot reciprocal (panel2 / G1 default; Engine F variant build)
O=gpurun_out/${1:-abpf}; mkdir -p $O
L=paper_2401_10089_b200/_build/liblogmpoly_b200.so
V=paper_2401_10089_b200/_build/var
for i in 1 2; do
echo "panel2 n=512" >> $O/r.txt; python tools/inv_bench.py 512 256 5 >> $O/r.txt 2>&1
echo "panel1 n=512" >> $O/r.txt; LGM_PANEL2=0 python tools/inv_bench.py 512 256 5 >> $O/r.txt 2>&1
for nn in 128 256; do
echo "g1 new n=$nn" >> $O/r.txt; python tools/inv_bench.py $nn 1024 5 >> $O/r.txt 2>&1
echo "g1 old n=$nn" >> $O/r.txt; LGM_LIB=$V/liblogmpoly_b200_g1old.so python tools/inv_bench.py $nn 1024 5 >> $O/r.txt 2>&1
done
for c in 2 1; do
echo "F base cfg $c" >> $O/r.txt; CFG=$c python tools/time_lib.py >> $O/r.txt 2>&1
echo "F pubfirst cfg $c" >> $O/r.txt; CFG=$c LGM_LIB=$V/liblogmpoly_b200_pubfirst.so python tools/time_lib.py >> $O/r.txt 2>&1
done
done
python tools/ab_grid.py 4 64 $L:LGM_PANEL2=0 $L > $O/ab.txt 2>&1
python tools/ab_grid.py 3b 256 $V/liblogmpoly_b200_g1old.so $L >> $O/ab.txt 2>&1
python tools/ab_grid.py 2 4096 $L $V/liblogmpoly_b200_pubfirst.so >> $O/ab.txt 2>&1
python tools/ab_grid.py 1 1 $L $V/liblogmpoly_b200_pubfirst.so >> $O/ab.txt 2>&1
cat $O/r.txt $O/ab.txt

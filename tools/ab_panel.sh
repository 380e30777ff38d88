# A/B: one barrier per pivot step in the G2 panels (LGM_PANEL_1BAR build) vs two
O=gpurun_out/abp; mkdir -p $O
V=paper_2401_10089_b200/_build/var
for i in 1 2; do
echo base >> $O/r.txt; python tools/inv_bench.py 512 256 5 >> $O/r.txt 2>&1
echo bar1 >> $O/r.txt; LGM_LIB=$V/liblogmpoly_b200_bar1.so python tools/inv_bench.py 512 256 5 >> $O/r.txt 2>&1
done
LGM_LIB=$V/liblogmpoly_b200_bar1.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bar1.csv python tools/inv_bench.py 512 256 1 > /dev/null 2>&1

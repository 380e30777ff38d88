#!/bin/bash
# inversion micro-benchmark + launch list + full ncu of the update / panel kernels
O=gpurun_out/${1:-inv}; mkdir -p $O
python tools/inv_bench.py 512 256 5 > $O/bench.txt 2>&1
python tools/inv_bench.py 4096 4 2 >> $O/bench.txt 2>&1
python tools/inv_bench.py 128 512 5 >> $O/bench.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches512.csv python tools/inv_bench.py 512 256 1 > /dev/null 2>&1
if [ "${2:-0}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gj_update2 --launch-skip 40 -c 2 -o $O/upd2 python tools/inv_bench.py 512 256 1 > $O/ncu_upd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gj_panel --launch-skip 20 -c 2 -o $O/panel python tools/inv_bench.py 512 256 1 > $O/ncu_panel.log 2>&1
fi
cat $O/bench.txt

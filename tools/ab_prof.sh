O=gpurun_out/ab2; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/inv_bench.py 512 256 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gj_update2_tma --launch-skip 17 -c 1 -o $O/tma python tools/inv_bench.py 512 256 1 > $O/ncu.log 2>&1

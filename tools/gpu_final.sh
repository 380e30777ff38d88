#!/bin/bash
# round-2 measurement session: full GPU suite, bench lines per config, reference arm, ncu
O=gpurun_out/${1:-final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=25 > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4.jsonl 2> $O/bench_cfg4.err
for c in 2 3 3b 1; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 >> $O/bench_other.jsonl 2>> $O/bench_other.err; done
timeout 1200 python bench.py --config 5b --steps 3 --warmup 3 --no-cpu-baseline >> $O/bench_other.jsonl 2>> $O/bench_other.err
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline >> $O/bench_other.jsonl 2>> $O/bench_other.err
timeout 900 python bench.py --max-k 9 --steps 10 --warmup 3 --no-cpu-baseline >> $O/bench_k9.jsonl 2>> $O/bench_other.err
timeout 900 python bench.py --config 2 --max-k 9 --steps 20 --warmup 5 --no-cpu-baseline >> $O/bench_k9.jsonl 2>> $O/bench_other.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_cfg4.jsonl 2> $O/ref_cfg4.err
for c in 2 3b 4 5b; do timeout 600 python tools/grid_phases.py $c >> $O/phases.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:logm_fused -c 1 -o $O/cfg2_fused python tools/prof_one.py 2 > $O/ncu_cfg2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_inv512.csv python tools/inv_bench.py 512 256 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gj_update2 --launch-skip 17 -c 1 -o $O/inv512_update2 python tools/inv_bench.py 512 256 1 > $O/ncu_upd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gj_panel_pair --launch-skip 9 -c 1 -o $O/inv512_panelpair python tools/inv_bench.py 512 256 1 > $O/ncu_panel.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_est512.csv python tools/est_bench.py 512 256 7 0 1 > /dev/null 2>&1
timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/graph_cfg4.csv python tools/prof_one.py 4 > $O/ncu_graph.log 2>&1
tail -3 $O/gputest.log

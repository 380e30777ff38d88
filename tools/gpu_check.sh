#!/bin/bash
# quick re-verification: GPU suite, config-4 bench line, inversion / estimator micro-benchmarks, phases
O=gpurun_out/${1:-chk}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.jsonl 2> $O/bench_cfg4.err
timeout 300 python tools/inv_bench.py 512 256 5 > $O/inv.txt 2>&1
timeout 300 python tools/est_bench.py 512 256 7 0 5 > $O/est.txt 2>&1
timeout 300 python tools/grid_phases.py 4 > $O/phases.txt 2>&1
if [ "${2:-tests}" = tests ]; then
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x --durations=10 > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
fi
cat $O/inv.txt $O/est.txt

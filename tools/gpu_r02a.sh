#!/bin/bash
# round-2 GPU session A: full GPU test suite, config-4 bench, compute-sanitizer passes
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench4.log 2>&1; echo "rc=$?" >> $O/bench4.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_probe.py > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_probe.py --quick > $O/racecheck.txt 2>&1; echo "rc=$?" >> $O/racecheck.txt
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_probe.py --quick > $O/synccheck.txt 2>&1; echo "rc=$?" >> $O/synccheck.txt
tail -3 $O/gputest.log $O/bench4.log

#!/bin/bash
# round-2 GPU session B: graph probe, Engine G device-driven control tests, config-4 bench
O=gpurun_out/r02b; mkdir -p $O
./tools/graph_cond_probe > $O/graph_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_abi.py -q -x -p no:cacheprovider -rf > $O/grid.log 2>&1; echo "rc=$?" >> $O/grid.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --deselect tests/test_gpu_configs.py::test_config5_as_written_status_parity > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench4.log 2>&1; echo "rc=$?" >> $O/bench4.log
tail -3 $O/grid.log $O/gputest.log $O/bench4.log

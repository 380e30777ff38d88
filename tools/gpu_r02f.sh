O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_schemes.py -q -p no:cacheprovider -rf > $O/schemes.log 2>&1; echo rc=$? >> $O/schemes.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x --deselect tests/test_gpu_configs.py::test_config5_as_written_status_parity --deselect tests/test_gpu_configs.py::test_config5b_one_matrix_vs_oracle > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench2.log 2>&1
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench4.log 2>&1

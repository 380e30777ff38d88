# Round-end bench sweep: every config's JSON line into gpurun_out/ (see profiles/bench_r01.jsonl)
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/b2.json 2>gpurun_out/b2.err
python bench.py --config 1 --steps 50 > gpurun_out/b1.json 2>gpurun_out/b1.err
python bench.py --config 3 --steps 10 > gpurun_out/b3.json 2>gpurun_out/b3.err
python bench.py --config 3b --steps 10 > gpurun_out/b3b.json 2>gpurun_out/b3b.err
python bench.py --config 4 --steps 5 > gpurun_out/b4.json 2>gpurun_out/b4.err
python bench.py --config 5b --steps 3 > gpurun_out/b5b.json 2>gpurun_out/b5b.err
python bench.py --config 5 --steps 3 --cpu-sample 1 > gpurun_out/b5.json 2>gpurun_out/b5.err
python bench.py --impl reference --steps 3 > gpurun_out/r2.json 2>gpurun_out/r2.err
tail -n 2 gpurun_out/*.err

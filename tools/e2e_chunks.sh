O=gpurun_out/e2e; mkdir -p $O
for c in 1 2 3 4; do echo "chunks $c" >> $O/r.txt; LGM_G_HOST_CHUNKS=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline >> $O/r.txt 2>&1; done

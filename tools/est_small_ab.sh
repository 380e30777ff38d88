O=gpurun_out/estf4; mkdir -p $O
for cfg in "65 256 7 1" "80 512 7 0" "96 512 7 0" "96 1024 8 1" "100 256 7 1" "128 1024 7 0"; do
  set -- $cfg
  EST_OUT=$O/a.npz LGM_EST_FUSED=0 timeout 300 python tools/est_bench.py $1 $2 $3 $4 5 >> $O/r.txt 2>&1
  EST_OUT=$O/b.npz timeout 300 python tools/est_bench.py $1 $2 $3 $4 5 >> $O/r.txt 2>&1
  python -c "
import numpy as np
a,b=np.load('$O/a.npz'),np.load('$O/b.npz')
print('$cfg','bitwise',np.array_equal(a['est'],b['est']),np.array_equal(a['passes'],b['passes']))" >> $O/r.txt
done
cat $O/r.txt
python -m pytest tests/test_gpu_grid.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2

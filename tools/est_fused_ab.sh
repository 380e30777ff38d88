#!/bin/bash
# A/B of the one-launch estimator (n <= 160), version 2 (default) against the per-step kernels
# (LGM_EST_FUSED=0) and against version 1 (-DEST_FUSED_V2=0 variant build): timing and bitwise
# estimates / pass counts over several n, powers and the product form; then config 3b.
O=gpurun_out/${1:-estf}; mkdir -p $O
L=paper_2401_10089_b200/_build/liblogmpoly_b200.so
V1=paper_2401_10089_b200/_build/var/liblogmpoly_b200_estv1.so
for cfg in "128 1024 7 0" "128 1024 8 1" "128 256 14 0" "96 512 7 0" "100 256 7 1" "130 256 7 0" "160 256 8 0" "65 256 7 1"; do
  set -- $cfg
  EST_OUT=$O/est_${1}_${2}_${3}_${4}_0.npz LGM_EST_FUSED=0 timeout 300 python tools/est_bench.py $1 $2 $3 $4 5 >> $O/est_ab.txt 2>&1
  EST_OUT=$O/est_${1}_${2}_${3}_${4}_1.npz timeout 300 python tools/est_bench.py $1 $2 $3 $4 5 >> $O/est_ab.txt 2>&1
  [ -f $V1 ] && LGM_LIB=$V1 timeout 300 python tools/est_bench.py $1 $2 $3 $4 5 >> $O/est_ab.txt 2>&1
  python - "$O" "$1_$2_$3_$4" >> $O/est_ab.txt 2>&1 <<'PY'
import sys, numpy as np
o, k = sys.argv[1], sys.argv[2]
a, b = np.load(f"{o}/est_{k}_0.npz"), np.load(f"{o}/est_{k}_1.npz")
print(k, "bitwise est:", np.array_equal(a["est"], b["est"]), "passes:", np.array_equal(a["passes"], b["passes"]),
      "max rel diff", float(np.max(np.abs(a["est"] - b["est"]) / np.abs(a["est"]))))
PY
done
python tools/ab_grid.py 3b 1024 $L:LGM_EST_FUSED=0 $L $V1 >> $O/est_ab.txt 2>&1
cat $O/est_ab.txt

#!/bin/bash
# A/B of the cluster-resident estimator (LGM_EST_CLUSTER=1) against the per-step kernels:
# timing and bitwise estimates / pass counts over several n, powers and the product form.
O=gpurun_out/${1:-estab}; mkdir -p $O
for cfg in "512 256 7 0" "512 256 8 1" "512 64 14 0" "448 128 7 0" "333 64 7 1" "257 64 7 0" "192 128 8 0"; do
  set -- $cfg
  for m in 0 1; do
    EST_OUT=$O/est_${1}_${2}_${3}_${4}_$m.npz LGM_EST_CLUSTER=$m timeout 300 python tools/est_bench.py $1 $2 $3 $4 5 >> $O/est_ab.txt 2>&1
  done
  python - "$O" "$1_$2_$3_$4" >> $O/est_ab.txt 2>&1 <<'PY'
import sys, numpy as np
o, k = sys.argv[1], sys.argv[2]
a, b = np.load(f"{o}/est_{k}_0.npz"), np.load(f"{o}/est_{k}_1.npz")
print(k, "bitwise est:", np.array_equal(a["est"], b["est"]), "passes:", np.array_equal(a["passes"], b["passes"]),
      "max rel diff", float(np.max(np.abs(a["est"] - b["est"]) / np.abs(a["est"]))))
PY
done
cat $O/est_ab.txt

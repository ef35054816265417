set -u
mkdir -p gpurun_out
for N in ${NS:-128 256}; do
  for k in 0 1; do
    GSE_CG_KEEP=$k KEEP_N=$N timeout 900 python scripts/cg_keep_ab.py > gpurun_out/keep_${N}_$k.json 2> gpurun_out/keep_${N}_$k.err
  done
done
echo done

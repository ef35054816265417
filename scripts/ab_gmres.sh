#!/bin/bash
# A/B of library variants on the GMRES(30) time (scripts/gmres_time.py, GM_N^3 conv-diff)
mkdir -p gpurun_out
for v in ${VARIANTS:-cur}; do
  if [ "$v" = cur ]; then unset GSE_LIB_PATH; else export GSE_LIB_PATH=$PWD/ab/$v.so; fi
  echo "== $v" >> gpurun_out/abgm_${ABTAG:-x}.txt
  timeout 600 python scripts/gmres_time.py >> gpurun_out/abgm_${ABTAG:-x}.txt 2>&1
done

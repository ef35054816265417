#!/bin/bash
# A/B of prebuilt library variants (ab/*.so vs the in-tree build) on the SpMV kernels.
mkdir -p gpurun_out
python -c "import paper_2411_04686_b200" 2>/dev/null
for v in ${VARIANTS:-cur old}; do
  if [ "$v" = cur ]; then unset GSE_LIB_PATH; else export GSE_LIB_PATH=$PWD/ab/$v.so; fi
  TAG=$v timeout 600 python scripts/spmv_ab.py >> gpurun_out/ab_${ABTAG:-x}.jsonl 2>> gpurun_out/ab_${ABTAG:-x}.err
done
unset GSE_LIB_PATH

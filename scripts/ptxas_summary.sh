#!/bin/bash
# usage: scripts/ptxas_summary.sh file.cu [regex]  -- registers / spills per kernel instantiation
f=$1; re=${2:-.}
cd /root/repo/paper_2411_04686_b200/csrc && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $GSE_NVCC_EXTRA -Xptxas -v -I ../../include -c $f -o ../build/$f.o 2>&1 | python3 -c "
import sys,re
cur=None
for l in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",l)
    if m: cur=m.group(1); continue
    m=re.search(r'(\d+) bytes spill stores',l)
    if m and cur: sp=m.group(1)
    m=re.search(r'Used (\d+) registers',l)
    if m and cur:
        if re.search('$re',cur): print(m.group(1),'regs', 'spill',sp, cur[:90])
        cur=None
"

set -u
mkdir -p gpurun_out
for v in ${VARIANTS:-p512 p1024 p2048}; do
  GSE_DEBUG=1 GSE_LIB_PATH=$PWD/ab/$v.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/r3_$v.json 2> gpurun_out/r3_$v.err
done
GSE_WIN_RING=0 GSE_LIB_PATH=$PWD/ab/p1024.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/r3_ring0.json 2> gpurun_out/r3_ring0.err
echo done

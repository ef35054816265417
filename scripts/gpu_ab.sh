mkdir -p gpurun_out
for v in t16 t32; do GSE_LIB_PATH=ab/$v.so MODES=win timeout 300 python scripts/win_ab.py > gpurun_out/winab_$v.json 2> gpurun_out/winab_$v.err; done
GSE_LIB_PATH=ab/t16.so PROF_MAT=powerlaw PROF_N=10000000 PROF_CG_ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,smsp__inst_executed.sum --clock-control none -k regex:k_spmv_win -c 4 --csv python scripts/prof_spmv.py > gpurun_out/ncu_m.csv 2>&1
echo done

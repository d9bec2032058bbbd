# ncu --set full of the patch apply (k_afw_apply_sc) inside the solve: 2 launches
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_afw_apply_sc' -c 2 -o /tmp/r02i_afw -f python profiles/prof_kernels.py --solve-iters 4 --only spmv --reps 1 > gpurun_out/r02i_ncu_afw.log 2>&1
ncu -i /tmp/r02i_afw.ncu-rep --page raw --csv > gpurun_out/r02i_ncu_afw_apply_sc.csv 2>/dev/null
ls -la gpurun_out/

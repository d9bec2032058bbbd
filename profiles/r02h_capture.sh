set -x
ncu --set full --clock-control none --import-source on -k regex:'k_afw_apply_sc|k_mf_spmv|k_pcg_pdir_afw2|k_nd_solve|k_coarse_restrict3c|k_pcg_update_r|k_coarse_gather' -o gpurun_out/r02h_iter3d -f python profiles/prof_kernels.py --solve-iters 4 --only spmv --reps 1 > gpurun_out/r02h_ncu_full.log 2>&1
ncu -i gpurun_out/r02h_iter3d.ncu-rep --page raw --csv > gpurun_out/r02h_ncu_iteration_3d.csv 2>/dev/null
ls -la gpurun_out/
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_bench_3d.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02h_bench_under_ncu.log 2>&1
tail -c 600 gpurun_out/r02h_bench_under_ncu.log
wc -l gpurun_out/r02h_launches_bench_3d.csv
gzip -f gpurun_out/r02h_launches_bench_3d.csv

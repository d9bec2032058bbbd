# final-state evidence, part 1: focused tests, bench, partitioned-path bench, ncu --set full of the iteration
set -x
python -m pytest tests -m gpu -q -x -k "coarse_weight or afw2 or solve_order" > gpurun_out/r02h_gpu_tests_subset.log 2>&1; tail -3 gpurun_out/r02h_gpu_tests_subset.log
python bench.py > gpurun_out/r02h_bench.log 2> gpurun_out/r02h_bench.err; tail -c 300 gpurun_out/r02h_bench.log; tail -5 gpurun_out/r02h_bench.err
timeout 600 python bench.py --force-comm --steps 2 --warmup 3 > gpurun_out/r02h_bench_force_comm.log 2> gpurun_out/r02h_bench_force_comm.err; tail -c 1500 gpurun_out/r02h_bench_force_comm.log; tail -5 gpurun_out/r02h_bench_force_comm.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_afw_apply_sc|k_mf_spmv|k_pcg_pdir_afw2|k_nd_solve|k_coarse_restrict3c|k_pcg_update_r|k_coarse_gather' -o /tmp/r02h_iter3d -f python profiles/prof_kernels.py --solve-iters 4 --only spmv --reps 1 > gpurun_out/r02h_ncu_full.log 2>&1
ncu -i /tmp/r02h_iter3d.ncu-rep --page raw --csv > gpurun_out/r02h_ncu_iteration_3d.csv 2>/dev/null
ls -la gpurun_out/ /tmp/r02h_iter3d.ncu-rep

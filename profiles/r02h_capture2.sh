# final-state evidence, part 2: full GPU test suite, bench, partitioned-path bench (one-rank NCCL), ncu launch list of one bench step
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02i_gpu_tests.log 2>&1; tail -3 gpurun_out/r02i_gpu_tests.log
python bench.py > gpurun_out/r02i_bench.log 2> gpurun_out/r02i_bench.err; tail -c 300 gpurun_out/r02i_bench.log; tail -5 gpurun_out/r02i_bench.err
timeout 400 python bench.py --force-comm --steps 2 --warmup 3 > gpurun_out/r02i_bench_force_comm.log 2> gpurun_out/r02i_bench_force_comm.err; tail -c 1500 gpurun_out/r02i_bench_force_comm.log; tail -5 gpurun_out/r02i_bench_force_comm.err
timeout 780 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file /tmp/r02i_launches.csv python bench.py --profile-run --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-other-configs > gpurun_out/r02i_bench_under_ncu.log 2>&1
wc -l /tmp/r02i_launches.csv
gzip -c /tmp/r02i_launches.csv > gpurun_out/r02i_launches_bench_3d.csv.gz
ls -la gpurun_out/

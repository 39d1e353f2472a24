set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fwd_kernel|lane_adj|lane_epi" -s 3 -c 3 -o gpurun_out/c3_kernels python tools/one_launch.py 4096 shadow22_dense blob128 > gpurun_out/ncu_full.log 2>&1
tail -c 600 gpurun_out/bench.json; tail -c 300 gpurun_out/bench_ref.json; tail -2 gpurun_out/ncu_full.log

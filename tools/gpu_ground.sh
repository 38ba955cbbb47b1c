# ground-removal (N2): parity tests, bench lines for G2/G3, launch list and one ncu --set full of k_g_count
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ground.py -x -q > gpurun_out/pytest_ground.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_ground.log
timeout 600 python bench.py --ground G3 --steps 10 --warmup 3 --check > gpurun_out/bench_ground_g3.json 2> gpurun_out/bench_ground_g3.err; echo g3=$?
timeout 600 python bench.py --ground G2 --steps 30 --warmup 5 --check > gpurun_out/bench_ground_g2.json 2> gpurun_out/bench_ground_g2.err; echo g2=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ground_g3.csv python bench.py --ground G3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ground.log 2>&1; echo ncu1=$?
if [ -n "$FULL" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_g_count -s 2 -c 1 -o gpurun_out/prof_ground_g3 python bench.py --ground G3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ground_full.log 2>&1; echo ncu2=$?; fi

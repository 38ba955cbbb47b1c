# Round profile: default bench line, launch list of the same command, ncu full capture of the top kernel.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu1=$?
python tools/prof_run.py C4 1.0 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_union_dense|k_dscatter|k_union_sparse" -s 4 -c 4 -o gpurun_out/prof_c4_full python tools/prof_run.py C4 1.0 2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

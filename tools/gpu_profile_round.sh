# Round profile: default bench line, reference arm, launch list of the bench command, ncu full
# capture of the dominant kernels (each ncu only after its command exited 0 without ncu).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref=$?
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu1=$?
python tools/prof_run.py C4 1.0 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_dcount|k_dscatter|k_dense_link|k_union_sparse|k_tail_stats|k_relabel}" -s ${SKIP:-7} -c ${COUNT:-7} -o gpurun_out/prof_c4_full python tools/prof_run.py C4 1.0 2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

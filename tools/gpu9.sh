python tools/prof_run.py C4 1.0 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 --csv --log-file gpurun_out/launches_c4.csv python tools/prof_run.py C4 1.0 2 > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:"k_dfixup|k_dcount|k_dscatter|k_union_dense" -s 8 -c 5 -o gpurun_out/prof_c4b python tools/prof_run.py C4 1.0 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu=$?

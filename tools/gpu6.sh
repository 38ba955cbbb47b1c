python tools/prof_run.py C5 1.0 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_union_sparse|k_dcount|k_dscatter|k_stats|k_relabel" -s 5 -c 5 -o gpurun_out/prof_c5 python tools/prof_run.py C5 1.0 2 > gpurun_out/ncu_c5.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_c5.log

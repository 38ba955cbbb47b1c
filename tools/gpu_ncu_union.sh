set -x
mkdir -p gpurun_out
python tools/prof_run.py C4 1.0 2 > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_union|k_dcount|k_cmark|k_dscatter" -s 8 -c 7 -o gpurun_out/prof_c4_union python tools/prof_run.py C4 1.0 2 > gpurun_out/ncu_c4u.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_c4u.log

# tests (filtered) + bench lines + launch lists
bash tools/gpu_r2_iter.sh
for C in ${LCONFS:-C4 C1}; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv python tools/prof_run.py $C 1.0 2 > gpurun_out/ncu_launch_$C.log 2>&1; echo launches_$C=$?
done

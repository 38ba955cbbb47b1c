# per-kernel launch list (ncu, cold-cache serialized) for one config; prints a summary
set -x
mkdir -p gpurun_out
C=${CONF:-C4}
python tools/prof_run.py $C 1.0 2 > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv python tools/prof_run.py $C 1.0 2 > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
python tools/launches.py gpurun_out/launches_$C.csv

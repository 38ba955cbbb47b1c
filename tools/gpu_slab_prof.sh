# per-rank profile of an emulated 8-way C4 slab step: stage times, ncu launch list, rank-time table
set -x
mkdir -p gpurun_out
C=${CONF:-C4}; W=${WORLD:-8}; R=${RANK:-3}
python tools/prof_slab.py $C $W $R > gpurun_out/prof_slab.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_slab.csv python tools/prof_slab.py $C $W $R > gpurun_out/ncu_slab.log 2>&1; echo ncu=$?
python tools/launches.py gpurun_out/launches_slab.csv
timeout 600 python tools/slab_rank_time.py $C 1,$W > gpurun_out/slab_rank.log 2>&1; echo rt=$?

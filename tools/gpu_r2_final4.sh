# Round-2 closing run, part 2: T6 schedule test, emulated slab rank times, launch lists of C1 and C5, batch/ground/AP lines.
set -x
O=gpurun_out/r02d; mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_schedules.py -q > $O/pytest_schedules.log 2>&1; echo sched=$?; tail -3 $O/pytest_schedules.log
timeout 900 python tools/slab_rank_time.py C4 1,2,4,8 > $O/slab_rank_C4.log 2>&1; echo rank_c4=$?
timeout 900 python tools/slab_rank_time.py C5 8 > $O/slab_rank_C5.log 2>&1; echo rank_c5=$?
cp gpurun_out/slab_rank_time_*.json $O/ 2>/dev/null
for C in C1 C5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$C.csv python tools/prof_run.py $C 1.0 2 > $O/ncu_launch_$C.log 2>&1; echo launches_$C=$?
done
timeout 600 python bench.py --batch 256 --check > $O/bench_batch_c2x256.json 2> $O/bench_batch.err; echo batch=$?
timeout 600 python bench.py --ground G3 --check > $O/bench_ground_g3.json 2> $O/bench_ground.err; echo ground=$?
timeout 600 python bench.py --ap --check > $O/bench_ap_voxel.json 2> $O/bench_ap.err; echo ap=$?

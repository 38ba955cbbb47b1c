# Mode B + async tests, C5 launch list, one C4/8 slab rank's launch list
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_async.py -x -q > gpurun_out/pytest_gpu_dist.log 2>&1; echo tests=$?; tail -3 gpurun_out/pytest_gpu_dist.log
python tools/prof_slab.py C4 8 3 > gpurun_out/prof_slab_plain.log 2>&1; echo slab_plain=$?; tail -2 gpurun_out/prof_slab_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_slab8.csv python tools/prof_slab.py C4 8 3 > gpurun_out/ncu_slab.log 2>&1; echo slab_launches=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python tools/prof_run.py C5 1.0 1 > gpurun_out/ncu_c5.log 2>&1; echo c5_launches=$?

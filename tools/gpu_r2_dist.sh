# Mode A/B GPU tests + emulated per-rank slab timing (C4, C5) + sanitizer
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_gpu_dist.log 2>&1; echo dist_tests=$?; tail -3 gpurun_out/pytest_gpu_dist.log
timeout 900 python tools/slab_rank_time.py C4 1,2,4,8 > gpurun_out/slab_rank_C4.log 2>&1; echo rank_c4=$?; tail -6 gpurun_out/slab_rank_C4.log
timeout 900 python tools/slab_rank_time.py C5 8 > gpurun_out/slab_rank_C5.log 2>&1; echo rank_c5=$?; tail -3 gpurun_out/slab_rank_C5.log
bash tools/gpu_sanitize.sh

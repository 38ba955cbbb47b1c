set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_gpu_dist.log 2>&1; echo pytest_dist=$?
tail -15 gpurun_out/pytest_gpu_dist.log
timeout 600 python bench.py --slab --steps 10 --warmup 3 --check --no-cpu-baseline > gpurun_out/bench_slab1.json 2> gpurun_out/bench_slab1.err; echo slab1=$?
cat gpurun_out/bench_slab1.json; tail -5 gpurun_out/bench_slab1.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log

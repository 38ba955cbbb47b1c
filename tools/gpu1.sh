set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --check > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bc2=$?
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bc4=$?
cat gpurun_out/smoke.log gpurun_out/bench_c2.json gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err

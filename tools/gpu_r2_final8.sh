# Round-2 closing run, last part: default bench line and the GPU suite on the final build (k_dinit one-wave grid).
set -x
O=gpurun_out/r02i; mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout 600 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench=$?
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_parity.py > $O/pytest_gpu_rest.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu_rest.log

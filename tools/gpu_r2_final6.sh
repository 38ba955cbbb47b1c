# Round-2 closing run, part 4: the new full-size forced-mode digest test, then the whole GPU suite as the driver runs it.
set -x
O=gpurun_out/r02f; mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k forced_grid_modes > $O/pytest_forced.log 2>&1; echo forced=$?; tail -15 $O/pytest_forced.log
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log

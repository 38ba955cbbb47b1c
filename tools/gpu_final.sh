# end-of-round validation: full GPU suite, smoke, default bench line + reference arm + profiles
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_final.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke.log
bash tools/gpu_profile_round.sh

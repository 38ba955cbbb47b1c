# parity + C4/C5 bench stage breakdown
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C4 C5}; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; tail -3 gpurun_out/bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac']); print({k: round(v,3) for k,v in d['stages_ms'].items()}); print({k:d['config'][k] for k in ('n_points','cells','components','pair_tests','dense_tests','group_pairs','dense_cells','dense_points')})"; done

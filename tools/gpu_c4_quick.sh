# C4 bench stage breakdown + 8-way slab rank stage times (no tests)
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo C4=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_C4.json')); print(d['value'], d['ms_per_step']); print({k: round(v,3) for k,v in d['stages_ms'].items()})"
python tools/prof_slab.py C4 8 3 2>&1 | tail -1

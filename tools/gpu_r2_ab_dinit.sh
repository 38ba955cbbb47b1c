# A/B of k_dinit's grid (one wave instead of four): C4 / C3 / C1 bench lines with --check, then the parity tests that reach k_dinit.
set -x
O=gpurun_out/r02h; mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
for c in C4 C3 C1 C4; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --check > $O/bench_$c.json 2> $O/bench_$c.err; echo $c=$?
  python -c "import json;d=json.loads(open('$O/bench_$c.json').read());print('$c',d['ms_per_step'],d.get('parity_bit_exact'))"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $O/pytest_parity.log 2>&1; echo parity=$?; tail -2 $O/pytest_parity.log

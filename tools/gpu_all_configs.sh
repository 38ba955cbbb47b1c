# bench line of every BASELINE config on the current build (parity checked for C1-C4)
mkdir -p gpurun_out
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --check > gpurun_out/bench_all_$c.json 2>/dev/null; echo $c=$?
done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_all_C5.json 2>/dev/null; echo C5=$?

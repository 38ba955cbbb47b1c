# refresh every judged bench line + the C4 profiles (after the kernel changes)
set -x
mkdir -p gpurun_out
bash tools/gpu_profile_round.sh
timeout 600 python bench.py --batch 256 --steps 10 --warmup 3 --check > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; echo batch=$?
timeout 600 python bench.py --ground G3 --steps 10 --warmup 3 --check > gpurun_out/bench_ground_g3.json 2> gpurun_out/bench_ground_g3.err; echo g3=$?
timeout 600 python bench.py --ground G2 --steps 30 --warmup 5 --check > gpurun_out/bench_ground_g2.json 2> gpurun_out/bench_ground_g2.err; echo g2=$?
timeout 600 python bench.py --ap --steps 10 --warmup 3 --check > gpurun_out/bench_ap.json 2> gpurun_out/bench_ap.err; echo ap=$?
timeout 900 python tools/slab_rank_time.py C4 1,2,4,8 > gpurun_out/slab_rank.log 2>&1; echo slab=$?

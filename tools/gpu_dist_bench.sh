# exercise bench.py's multi-rank slab path on ONE GPU (gloo exchange; both ranks on cuda:0)
set -x
mkdir -p gpurun_out
export FEC_DIST_BACKEND=gloo FEC_FORCE_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --check --config ${CONF:-C3} > gpurun_out/bench_dist2.json 2> gpurun_out/bench_dist2.err; echo dist2=$?
cat gpurun_out/bench_dist2.json; tail -5 gpurun_out/bench_dist2.err

# Round-2 closing run, part 5: bench.py's N>1 launch path on one GPU (gloo exchange, both ranks on cuda:0; not a bench value),
# the reference arm under torchrun, the slab path at N=1.
set -x
O=gpurun_out/r02g; mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
export FEC_DIST_BACKEND=gloo FEC_FORCE_DEVICE=0
for C in C3 C4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --check --config $C > $O/bench_dist2_$C.json 2> $O/bench_dist2_$C.err; echo dist2_$C=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/bench_ref_dist2.json 2> $O/bench_ref_dist2.err; echo refdist2=$?
unset FEC_DIST_BACKEND FEC_FORCE_DEVICE
timeout 600 python bench.py --slab --check --no-cpu-baseline > $O/bench_slab1.json 2> $O/bench_slab1.err; echo slab1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err; echo torchrun1=$?

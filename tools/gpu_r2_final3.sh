# Round-2 closing run (after 558d7e3 / 4bf47fc / 5f77c8f): GPU suite, smoke, default bench line (C4) +
# reference arm, every config, ncu launch list of the bench command, ncu --set full of the C4 kernels.
set -x
O=gpurun_out/r02c; mkdir -p $O/configs
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/nvsmi.txt
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench=$?
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err; echo ref=$?
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --check > $O/configs/bench_$c.json 2> $O/configs/bench_$c.err; echo $c=$?
done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > $O/configs/bench_C5.json 2> $O/configs/bench_C5.err; echo C5=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1; echo ncu_launch_c4=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_bbox|k_cmark|k_dcount2|k_dcomps|k_dscatter|k_dense_link|k_union_sparse_local|k_dense_items|k_relabel_in" -s 11 -c 11 -o $O/ncu_c4_full python tools/prof_run.py C4 1.0 2 > $O/ncu_c4_full.log 2>&1; echo ncu_full_c4=$?

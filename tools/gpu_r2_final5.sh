# Round-2 closing run, part 3: 10,000 random clouds x 4 grid modes vs the oracle on the final build; ncu --set full of C5's top kernels.
set -x
O=gpurun_out/r02e; mkdir -p $O
python -c "import sys; sys.path.insert(0,'.'); from paper_2208_07678_b200.build import build; build()" || exit 1
timeout 900 python tools/stress_parity.py 10000 > $O/stress_parity.log 2>&1; echo stress=$?; cp gpurun_out/stress_parity.json $O/
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_union_sparse$|k_sgather|k_onesweep|k_relabel_b1|k_relabel_b2c|k_tail_stats" -c 9 -o $O/ncu_c5_full python tools/prof_run.py C5 1.0 1 > $O/ncu_c5_full.log 2>&1; echo ncu_full_c5=$?

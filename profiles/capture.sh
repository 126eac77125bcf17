#!/bin/bash
# Round capture recipe run on the GPU box (gpurun): tests, smoke, bench, then the ncu passes.
# ncu passes run only after the same command exited 0 without ncu.
set -u
R=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$R.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_$R.log 2>&1
python bench.py > $O/bench_$R.log 2>&1
echo "bench rc=$?" >> $O/bench_$R.log
# cfg2 CG step: launch list (serialised, cold per launch) and one full capture of the three CG kernels
python bench.py --steps 1 --warmup 3 --no-cpu --no-scale > $O/bench_short_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-scale > $O/ncu_launch_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_t8|k_update_r|k_update_px" -c 3 \
    -o $O/full_$R -f python bench.py --steps 1 --warmup 3 --no-cpu --no-scale > $O/ncu_full_$R.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full_$R.log
# cfg1 level-3 correction step: launch list and the inner-sweep kernels
python tests/diag_step3.py 3 2 > $O/diag_step3_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_$R.csv \
    python tests/diag_step3.py 3 1 > $O/ncu_step_launch_$R.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"tridiag|arrow_eig|arrow_vec|orbital_border|k_select|hartree_delta|k_gemm" -c 7 \
    -o $O/inner_$R -f python tests/diag_step3.py 3 1 > $O/ncu_inner_$R.log 2>&1
echo "ncu rc=$?" >> $O/ncu_inner_$R.log

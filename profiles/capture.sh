#!/bin/bash
# Round capture recipe run on the GPU box (gpurun): tests, smoke, bench, then the ncu passes.
# ncu passes run only after the same bench command exited 0 without ncu.
set -u
R=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$R.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_$R.log 2>&1
python bench.py > $O/bench_$R.log 2>&1
rc=$?
echo "bench rc=$rc" >> $O/bench_$R.log
python bench.py --steps 1 --warmup 3 --no-cpu > $O/bench_short_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_launch_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_dot|k_update_xr|k_update_p" -c 3 \
    -o $O/full_$R -f python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full_$R.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full_$R.log

#!/bin/bash
# configs[3] (N = 21) on a reduced adaptive hierarchy: ncu --set full of the multi-column CG kernels (row SpMM with
# the shift operator, residual and direction updates), with and without the union-tile view for 8 lanes per tile
set -u
T=${1:-r02k}
O=gpurun_out
mkdir -p $O
K='k_spmm_dot|k_spmm_ut|k_update_r|k_update_px'
KSB_PROBE_FAMILIES=0 timeout 900 ncu --kernel-id "::regex:^($K)\$:40" --set full --clock-control none --import-source on \
    -o $O/n21_row_$T -f python profiles/adaptive_probe.py cfg4 ${2:-1.5e6} > $O/ncu_n21_row_$T.log 2>&1
KSB_SPMM_UT=2 KSB_PROBE_FAMILIES=0 timeout 900 ncu --kernel-id "::regex:^($K)\$:40" --set full --clock-control none --import-source on \
    -o $O/n21_ut_$T -f python profiles/adaptive_probe.py cfg4 ${2:-1.5e6} > $O/ncu_n21_ut_$T.log 2>&1
python profiles/summarize.py full $O/n21_row_$T.ncu-rep $O/n21_ut_$T.ncu-rep > $O/n21_${T}_ncu_full.txt 2>&1
for x in row ut; do
  ncu -i $O/n21_${x}_$T.ncu-rep --page source --csv 2>/dev/null | gzip > $O/n21_${x}_${T}_source.csv.gz
done
rm -f $O/n21_row_$T.ncu-rep $O/n21_ut_$T.ncu-rep

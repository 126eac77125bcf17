#!/bin/bash
# ncu --set full of the union-tile wide SpMM (one launch without and one with the shift operator) inside an
# N = 120 correction step on the 2.05 M-DOF uniform level; summary + per-line source page come back as text.
set -u
T=${1:-r02g}
O=gpurun_out
mkdir -p $O
timeout 900 ncu --kernel-id "::regex:^k_spmm_ut\$:3" --set full --clock-control none --import-source on \
    -o $O/ut_a_$T -f python profiles/phase_probe.py ${2:-4} 120 1 > $O/ncu_ut_$T.log 2>&1
timeout 900 ncu --kernel-id "::regex:^k_spmm_ut\$:20" --set full --clock-control none --import-source on \
    -o $O/ut_b_$T -f python profiles/phase_probe.py ${2:-4} 120 1 >> $O/ncu_ut_$T.log 2>&1
python profiles/summarize.py full $O/ut_a_$T.ncu-rep $O/ut_b_$T.ncu-rep > $O/ut_${T}_ncu_full.txt 2>&1
for x in a b; do
  ncu -i $O/ut_${x}_$T.ncu-rep --page source --csv 2>/dev/null | gzip > $O/ut_${x}_${T}_source.csv.gz
  ncu -i $O/ut_${x}_$T.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/ut_${x}_${T}_raw.csv.gz
done
ls -la $O/*.ncu-rep
rm -f $O/ut_a_$T.ncu-rep $O/ut_b_$T.ncu-rep

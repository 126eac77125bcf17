#!/bin/bash
# ncu --set full of the union-tile SpMM on configs[4]'s adaptive hierarchy (N = 120) at a reduced size
set -u
T=${1:-r02n}
O=gpurun_out
mkdir -p $O
KSB_PROBE_FAMILIES=0 timeout 1200 ncu --kernel-id "::regex:^(k_spmm_ut|k_update_r|k_update_px|k_trueres)\$:12" --set full --clock-control none \
    --import-source on -o $O/uta_$T -f python profiles/adaptive_probe.py cfg5 ${2:-2e6} > $O/ncu_uta_$T.log 2>&1
python profiles/summarize.py full $O/uta_$T.ncu-rep > $O/uta_${T}_ncu_full.txt 2>&1
ncu -i $O/uta_$T.ncu-rep --page source --csv 2>/dev/null | gzip > $O/uta_${T}_source.csv.gz
rm -f $O/uta_$T.ncu-rep

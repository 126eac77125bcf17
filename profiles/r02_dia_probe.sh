#!/bin/bash
# ncu --set full of cfg2 SpMM variants, summarised on the box (reports are too big to bring back)
for v in "KSB_DIA_Z=8,KSB_DIA_ZC=4:k_spmm_dia_z" "KSB_DIA_Z=0:k_spmm_dia_tv"; do
  e=${v%%:*}; k=${v##*:}; tag=$(echo $e | tr '=,' '__')
  env $(echo $e | tr ',' ' ') timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 --launch-skip 2 -f \
      -o /tmp/rep_$tag python profiles/cfg2_probe.py 3 > gpurun_out/ncu_$tag.log 2>&1; echo ncu $e $?
  python profiles/summarize.py full /tmp/rep_$tag.ncu-rep > gpurun_out/sum_$tag.txt 2>&1
  ncu -i /tmp/rep_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$tag.csv 2>/dev/null
done

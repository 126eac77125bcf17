#!/bin/bash
# CUDA-event times of the cfg2 SpMM variants (50 fixed-count CG iterations, profiles/cfg2_probe.py --time), then an
# ncu --set full capture of the default kernel, summarised on the box
python -m pytest tests/test_gpu_dia.py tests/test_gpu_scale.py -m gpu -q -x -k "dia or stencil or cfg2 or t8" 2>&1 | tail -3
for v in "KSB_DIA_ZW=1" "KSB_DIA_ZW=0" "KSB_DIA_ZT=0" "KSB_SPMM_DIA=0"; do
  echo "== $v"; env $v python profiles/cfg2_probe.py 3 --time 2>&1 | grep -E "spmm|Error|error"
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_dia_zw -c 1 --launch-skip 2 -f -o /tmp/rep_zt python profiles/cfg2_probe.py 3 > gpurun_out/ncu_zt.log 2>&1; echo ncu $?
python profiles/summarize.py full /tmp/rep_zt.ncu-rep > gpurun_out/sum_zt.txt 2>&1
ncu -i /tmp/rep_zt.ncu-rep --page source --csv --print-source sass > gpurun_out/src_zt.csv 2>/dev/null

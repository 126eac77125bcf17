#!/bin/bash
# CUDA-event times of the cfg2 SpMM variants (50 fixed-count CG iterations, profiles/cfg2_probe.py --time)
for v in "KSB_DIA_Z=0" "KSB_DIA_Z=0 KSB_DIA_MINB=3" "KSB_DIA_Z=0 KSB_DIA_TV=0 KSB_DIA_PF=0"; do
  echo "== $v"; env $v python profiles/cfg2_probe.py 3 --time 2>&1 | grep -E "spmm|Error|error"
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv

#!/bin/bash
# A/B of the stencil (DIA) SpMM lane-group variants against the T8 kernel on the cfg2 bench (GPU box).
python -m pytest tests/test_gpu_dia.py tests/test_gpu_scale.py -m gpu -q -x -k "dia or stencil or cfg2 or t8" > gpurun_out/pt_dia.log 2>&1; tail -3 gpurun_out/pt_dia.log
for v in "KSB_SPMM_DIA=0" "KSB_DIA_G=16" "KSB_DIA_G=8" "KSB_DIA_G=4"; do
  env $v python bench.py --steps 3 --warmup 3 --no-cpu --no-scale --no-parity > gpurun_out/b_ab.log 2>&1
  echo "$v"; python -c "
import json; d=json.loads(open('gpurun_out/b_ab.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['cg_update_r_avg_ms'], d['cg_update_px_avg_ms'], d['clocks'])" || tail -5 gpurun_out/b_ab.log
done

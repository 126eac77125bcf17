#!/bin/bash
# A/B of the SpMM variants on the cfg2 bench (GPU box): pytest -m gpu, then bench per variant.
python -m pytest tests -m gpu -q -x > gpurun_out/pt_ab.log 2>&1; tail -2 gpurun_out/pt_ab.log
for v in "$@"; do
  env $v python bench.py --steps 3 --warmup 3 --no-cpu --no-scale > gpurun_out/b_ab.log 2>&1
  echo "$v"; python -c "
import json; d=json.loads(open('gpurun_out/b_ab.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['cg_update_r_avg_ms'], d['cg_update_px_avg_ms'])"
done

#!/bin/bash
# A/B of environment variants on the cfg1 level-3 correction step (tests/diag_step3.py)
for v in "$@"; do
  env $v python tests/diag_step3.py 3 4 > gpurun_out/ab_step.log 2>&1
  echo "$v: $(grep '"step": 3' gpurun_out/ab_step.log)"
done

#!/bin/bash
# A/B of the wide (N = 120) SpMM on the cfg5-like scale step (GPU box): "SYNC LD [DIE [REORDER [WIDE [MINB]]]]" tuples.
for v in "$@"; do
  set -- $v
  echo "SYNC=$1 LD=$2 DIE=${3:-0} REORDER=${4:-1} WIDE=${5:-1} MINB=${6:-4}"
  KSB_SPMM_MINB=${6:-4} KSB_SPMM_WIDE=${5:-1} KSB_CG_REORDER=${4:-1} KSB_SPMM_DIE=${3:-0} KSB_SPMM_SYNC=$1 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tests')
import diag_scale as d
from paper_2103_02824_b200.workloads import sphere_atoms
d.run('cfg5-like N=120, 2.1M dofs', sphere_atoms(), 120, 30.0, 4, 10, steps=1, profile=True, ld=$2)
" 2>&1 | grep -E "spmm|cg_update|ms_total|name" | cut -c1-300
done

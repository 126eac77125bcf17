#!/bin/bash
# Same-box A/B of prebuilt libraries: copy ab_libs/libksb_<tag>.so over the in-tree library, run the short cfg2 +
# correction-step bench, print (tag, ms/step, SpMM ms, update_r ms, update_px ms, SM MHz). Usage: bash profiles/ab_lib.sh old new old new
for v in "$@"; do
  cp ab_libs/libksb_$v.so paper_2103_02824_b200/_lib/libksb.so
  python bench.py --steps 3 --warmup 3 --no-cpu --no-scale > gpurun_out/b_ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/b_ab_$v.log').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), round(d['roofline']['avg_launch_ms'],4), round(d['cg_update_r_avg_ms'],4), round(d['cg_update_px_avg_ms'],4), d['clocks']['sm_mhz'])"
done

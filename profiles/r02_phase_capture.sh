#!/bin/bash
# Per-phase evidence for one N = 120 correction step on the 2.05 M-DOF uniform level (and cfg1-size N = 1):
# CUDA-event family times (phase_probe.py), then -- only after that run exited 0 -- an ncu launch list and one
# `--set full` capture of the second invocation of every kernel of the step.
set -u
T=${1:-r02f}
O=gpurun_out
mkdir -p $O
if [ "${SKIP_PROBE:-0}" != "1" ]; then
python profiles/phase_probe.py 4 120 2 > $O/phase_${T}_n120.json 2> $O/phase_${T}_n120.err || { echo "probe failed"; tail -5 $O/phase_${T}_n120.err; exit 1; }
python profiles/phase_probe.py 3 1 2 > $O/phase_${T}_n1.json 2> $O/phase_${T}_n1.err
fi
K='k_elem_mass|k_elem_stiffness|k_gather|k_axpby|k_rho_vxc|k_moments1|k_moments2|k_sqload_elem|k_sqload_elem_warp|k_gather_vinc|k_gather_vinc_rows|k_xc_field|k_lift|k_expand|k_norm_parts|k_energy_parts|k_mg_smooth|k_mg_restrict|k_mg_prolong_add|k_pcg_spmv_dot|k_pcg_axpy|k_spmm_dot|k_spmm_ut|k_spmm_dia|k_update_r|k_update_px|k_trueres|k_proj_shared|k_proj_orbital_wide|k_proj_fold|k_min_diag|k_permute_rows|k_init|k_full_from|k_coarse_mat|k_coarse_vec'
timeout 1500 ncu --kernel-id "::regex:^($K)\$:2" --set full --clock-control none --import-source on \
    -o $O/phase_${T}_n120 -f python profiles/phase_probe.py 4 120 1 > $O/ncu_phase_${T}.log 2>&1
echo "ncu rc=$?" >> $O/ncu_phase_${T}.log
# the report (with sources) is too large to bring back: keep the text summary and the raw csv page
python profiles/summarize.py full $O/phase_${T}_n120.ncu-rep > $O/phase_${T}_n120_ncu_full.txt 2>&1
ncu -i $O/phase_${T}_n120.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/phase_${T}_n120_raw.csv.gz
rm -f $O/phase_${T}_n120.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_phase_${T}.csv \
    python profiles/phase_probe.py 4 120 1 > $O/ncu_phase_launch_${T}.log 2>&1
echo "ncu rc=$?" >> $O/ncu_phase_launch_${T}.log

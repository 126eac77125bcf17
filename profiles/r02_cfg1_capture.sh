#!/bin/bash
# cfg1 level-3 correction step (N = 1, 250,047 rows): ncu --set full of the single-column cooperative CG, the Hartree
# multigrid kernels and the inner-sweep kernels (L2 hit rates: the 49 MB operator is L2-resident)
set -u
T=${1:-r02u}
O=gpurun_out
mkdir -p $O
python tests/diag_step3.py 3 2 > $O/diag_step3_$T.log 2>&1 || exit 1
K='k_cg_coop|k_mg_smooth|k_pcg_spmv_dot|k_tridiag_cluster|k_arrow_eig|k_arrow_vec|k_select|k_border_q|k_proj_shared|k_proj_orbital|k_elem_mass|k_elem_stiffness|k_gather|k_rho_vxc|k_sqload_elem'
timeout 900 ncu --kernel-id "::regex:^($K)\$:2" --set full --clock-control none -o $O/cfg1_$T -f \
    python tests/diag_step3.py 3 2 > $O/ncu_cfg1_$T.log 2>&1
echo "ncu rc=$?" >> $O/ncu_cfg1_$T.log
python profiles/summarize.py full $O/cfg1_$T.ncu-rep > $O/cfg1_${T}_ncu_full.txt 2>&1
rm -f $O/cfg1_$T.ncu-rep

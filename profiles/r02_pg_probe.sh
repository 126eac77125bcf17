timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_proj_gemm -c 1 --launch-skip 1 -f -o /tmp/rep_pg python profiles/proj_probe.py 2e5 > gpurun_out/ncu_pg.log 2>&1; echo ncu $?
python profiles/summarize.py full /tmp/rep_pg.ncu-rep > gpurun_out/sum_pg.txt 2>&1
ncu -i /tmp/rep_pg.ncu-rep --page source --csv --print-source sass > gpurun_out/src_pg.csv 2>/dev/null

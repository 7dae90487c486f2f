# ncu source-level (cuda,sass) export of the C5 n=4 sweeps: where the shared-memory bank conflicts are
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mid -c 5 -o /tmp/r4f_c5n4 python tools/profile_solve.py --config c5n4 --solves 1 > gpurun_out/r4f_ncu_c5n4.log 2>&1
ncu -i /tmp/r4f_c5n4.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip -9 > gpurun_out/r4f_c5n4_source.csv.gz
ls -la gpurun_out/r4f*

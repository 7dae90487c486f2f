# ncu source-level (cuda,sass) export of the C5 n=4 sweeps: where the shared-memory bank conflicts are
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mid -c 5 -o /tmp/r4j_c5n4 python tools/profile_solve.py --config c5n4 --solves 1 > gpurun_out/r4j_ncu_c5n4.log 2>&1
ncu -i /tmp/r4j_c5n4.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip -9 > gpurun_out/r4j_c5n4_source.csv.gz
ncu -i /tmp/r4j_c5n4.ncu-rep --page raw --csv > gpurun_out/r4j_c5n4_raw.csv 2>/dev/null
SFEM_LIB= timeout 200 python tools/check_configs.py c5n1 c5n2 c5n4 c5n9 c3 > gpurun_out/r4j_configs.txt 2>&1

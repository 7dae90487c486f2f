# ncu --set full captures of the C2 line kernel (sweep_mid_gw) and the C5 n=4 strided / fused sweeps
mkdir -p gpurun_out
timeout 300 python tools/lines_times.py > gpurun_out/r1n_c2_lines_times.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_mid_gw -c 1 -o gpurun_out/r1n_c2 python tools/lines_times.py > gpurun_out/r1n_ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mid -c 3 -o gpurun_out/r1n_c5n4 python tools/profile_solve.py --config c5n4 --solves 1 > gpurun_out/r1n_ncu_c5n4.log 2>&1

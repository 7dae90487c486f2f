mkdir -p gpurun_out
for c in c5n1 c5n2 c5n4; do
  echo "== $c" >> gpurun_out/r1m2_ab.txt
  timeout 600 python tools/kernel_times.py --config $c --reps 5 --rounds 3 variants/mixg2.so paper_1701_03967_b200/libsfem_b200.so >> gpurun_out/r1m2_ab.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1m2_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1m2_pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_mid -c 3 -o gpurun_out/r1m2_c3 python tools/profile_solve.py --config c3 --solves 1 > gpurun_out/r1m2_ncu_c3.log 2>&1

# A/B of the mid-kernel tile load/store unrolling (SFEM_MID_UNROLL 1 / 4 / 8 = default)
mkdir -p gpurun_out
for c in c3 c5n1 c5n2 c5n4 c5n9; do
  echo "== $c" >> gpurun_out/r1m4_unroll_ab.txt
  timeout 600 python tools/kernel_times.py --config $c --reps 5 --rounds 3 variants/unroll1.so variants/unroll4.so paper_1701_03967_b200/libsfem_b200.so >> gpurun_out/r1m4_unroll_ab.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1m4_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1m4_pytest_gpu.log
timeout 600 python tools/shape_survey.py > gpurun_out/r1m4_shapes.txt 2>&1
timeout 600 python tools/shape_survey_k.py > gpurun_out/r1m4_shapes_k.txt 2>&1

# A/B of the mid-kernel mix item width (SFEM_MID_MIXG 1 vs 2) on C3 / C5, then parity of the default build
mkdir -p gpurun_out
for c in c3 c5n1 c5n2 c5n4 c5n9; do
  echo "== $c" >> gpurun_out/r1m_mixg_ab.txt
  timeout 600 python tools/kernel_times.py --config $c --reps 5 --rounds 3 variants/mixg1.so variants/mixg2.so >> gpurun_out/r1m_mixg_ab.txt 2>&1
done
SFEM_LIB=variants/mixg1.so timeout 600 python tools/shape_survey.py > gpurun_out/r1m_shapes_mixg1.txt 2>&1
SFEM_LIB=variants/mixg2.so timeout 600 python tools/shape_survey.py > gpurun_out/r1m_shapes_mixg2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1m_pytest_gpu_mixg2.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1m_pytest_gpu_mixg2.log

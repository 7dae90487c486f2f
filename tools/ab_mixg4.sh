mkdir -p gpurun_out
for c in c5n1 c5n2 c5n4; do
  echo "== $c" >> gpurun_out/r1m_mixg4_ab.txt
  timeout 600 python tools/kernel_times.py --config $c --reps 5 --rounds 3 variants/mixg2.so variants/mixg4.so >> gpurun_out/r1m_mixg4_ab.txt 2>&1
done
SFEM_LIB=variants/mixg4.so timeout 600 python tools/shape_survey.py > gpurun_out/r1m_shapes_mixg4.txt 2>&1

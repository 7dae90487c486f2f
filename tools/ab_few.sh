# A/B of the radix-16 plan rule for the general-shape mid kernels (SFEM_MID_FEW_RULE 0 = default vs 1)
mkdir -p gpurun_out
for lib in paper_1701_03967_b200/libsfem_b200.so variants/few1.so; do
  echo "== $lib" >> gpurun_out/r1m5_few_ab.txt
  SFEM_LIB=$lib timeout 600 python tools/shape_survey.py >> gpurun_out/r1m5_few_ab.txt 2>&1
  SFEM_LIB=$lib timeout 600 python tools/shape_survey_k.py >> gpurun_out/r1m5_few_ab.txt 2>&1
done

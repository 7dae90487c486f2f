mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "mid_kernels" > gpurun_out/r1m3_pytest_mid.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1m3_pytest_mid.log
timeout 600 python tools/shape_survey_k.py > gpurun_out/r1m3_shapes_k.txt 2>&1
timeout 600 python tools/shape_survey.py > gpurun_out/r1m3_shapes.txt 2>&1

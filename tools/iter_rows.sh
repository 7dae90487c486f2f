# Iteration check for the fused row kernel: A/B times, bitwise parity test,
# one ncu --set full of both kernels.  P=<tag> bash tools/iter_rows.sh
P=${P:-r2x}
mkdir -p gpurun_out
timeout 200 python tools/rows_ab.py > gpurun_out/${P}_rows_ab.txt 2>&1
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "rows_fused or fast_kernels or fast_3d" > gpurun_out/${P}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${P}_pytest.log
if [ -z "$NO_NCU" ]; then
python tools/rows_ab.py once && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sweep_rows_fused|sweep_bulk_rows" -c 2 -o gpurun_out/${P}_rows python tools/rows_ab.py once > gpurun_out/${P}_ncu.log 2>&1
fi

# Round-2 GPU check: FP64 probe, pytest -m gpu, smoke, bench (ours + reference arm).
P=${P:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt 2>&1
nproc >> gpurun_out/${P}_smi.txt; free -g >> gpurun_out/${P}_smi.txt
if [ -z "$SKIP_PROBE" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_probe tools/fp64_probe.cu && timeout 120 /tmp/fp64_probe > gpurun_out/${P}_fp64_probe.txt 2>&1
fi
timeout ${PYT_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYT_ARGS} > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/${P}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${P}_bench_c4.json 2> gpurun_out/${P}_bench_c4.err
if [ -z "$SKIP_REF" ]; then
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
fi
echo done

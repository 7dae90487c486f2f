# Round-end GPU check: pytest -m gpu, smoke, bench (ours + reference arm), the
# ncu launch list of the bench command and one ncu --set full of the dominant
# kernel.  P=<tag> bash tools/r2_final.sh
P=${P:-r3z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/${P}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${P}_bench_c4.json 2> gpurun_out/${P}_bench_c4.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-configs --e2e-steps 2 > gpurun_out/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_rows_fused -s 3 -c 1 -o gpurun_out/${P}_fused python bench.py --steps 3 --warmup 3 --no-cpu --no-configs --e2e-steps 2 > gpurun_out/${P}_ncu_full.log 2>&1
echo done

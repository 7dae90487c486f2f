# A/B of discarding dead global FFT work slices in the C2 line kernel (sweep_mid_gw)
mkdir -p gpurun_out
for lib in variants/nodiscard.so paper_1701_03967_b200/libsfem_b200.so; do
  for r in 1 2; do echo "== $lib" >> gpurun_out/r1n_discard_ab.txt; SFEM_LIB=$lib timeout 300 python tools/lines_times.py >> gpurun_out/r1n_discard_ab.txt 2>&1; done
done
timeout 900 python -m pytest tests -m gpu -q -k "config2 or mid_kernels or 1d or lines or roundtrip" > gpurun_out/r1n_pytest_discard.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1n_pytest_discard.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep_mid_gw -c 3 --csv python tools/lines_times.py > gpurun_out/r1n_discard_dram.csv 2>&1

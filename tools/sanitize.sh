# compute-sanitizer over the small cases of tools/sanitize_cases.py
# (racecheck / synccheck / memcheck over the mbarrier / TMA /
# bulk-copy kernels and the peer loopback).  P=<tag> bash tools/sanitize.sh
P=${P:-r2s}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_cases.py > gpurun_out/${P}_cases_plain.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_cases_plain.log
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_TIMEOUT:-1200} $CS --tool $tool --print-limit 30 --error-exitcode 9 \
      python tools/sanitize_cases.py ${SAN_CASES} > gpurun_out/${P}_sanitizer_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${P}_sanitizer_${tool}.log
done
echo sanitize done

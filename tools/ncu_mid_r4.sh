# ncu --set full captures of the current mid kernels: C3 (3 sweeps), C5 n=4 and n=9 (5 sweeps each), C2 line ops.
# The reports are exported to raw csv on the box (gpurun_out is capped at 64 MiB); C3's source page is kept gzipped.
mkdir -p gpurun_out
for c in c3 c5n4 c5n9; do
  timeout 300 python tools/profile_solve.py --config $c --solves 2 > gpurun_out/r4d_${c}_plain.txt 2>&1 || exit 1
done
timeout 300 python tools/lines_times.py > gpurun_out/r4d_c2_lines_times.txt 2>&1
cap() {  # name count command...
  local name=$1 cnt=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_mid -c $cnt -o /tmp/r4d_$name "$@" > gpurun_out/r4d_ncu_$name.log 2>&1
  ncu -i /tmp/r4d_$name.ncu-rep --page raw --csv > gpurun_out/r4d_${name}_raw.csv 2>/dev/null
}
cap c3 3 python tools/profile_solve.py --config c3 --solves 1
ncu -i /tmp/r4d_c3.ncu-rep --page source --csv 2>/dev/null | gzip -9 > gpurun_out/r4d_c3_source.csv.gz
cap c5n4 5 python tools/profile_solve.py --config c5n4 --solves 1
cap c5n9 5 python tools/profile_solve.py --config c5n9 --solves 1
cap c2 3 python tools/lines_times.py
ls -la gpurun_out /tmp/r4d_* > gpurun_out/r4d_ls.txt

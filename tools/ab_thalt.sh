# A/B of the C5 tile thread counts (n=1: 512 -> 256; n=2, 4, 9: 256 -> 512)
mkdir -p gpurun_out
for c in c5n1 c5n2 c5n4 c5n9; do
  echo "== $c" >> gpurun_out/r1o_thalt_ab.txt
  timeout 600 python tools/kernel_times.py --config $c --reps 5 --rounds 3 paper_1701_03967_b200/libsfem_b200.so variants/thalt.so >> gpurun_out/r1o_thalt_ab.txt 2>&1
done

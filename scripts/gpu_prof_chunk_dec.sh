# ncu --set full of the decoder (K4) at chunk 1024 vs 65536, 2^28 BF16 words
for c in 1024 65536; do
  timeout 600 ncu -f --set full --clock-control none -k regex:decode_persistent -s 1 -c 1 \
    -o gpurun_out/prof_dec_c$c python scripts/profile_kernels.py bf16 $((1<<28)) 2 4 $c > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep

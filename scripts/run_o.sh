O=gpurun_out
for v in default r01; do
  if [ "$v" = default ]; then L=""; else L="SNAP_B200_LIB=paper_1111_5572_b200/lib/variants/libsnapb200_$v.so"; fi
  env $L timeout 900 ncu --set full --clock-control none -k 'regex:align_kernel' -c 1 -o $O/prof_c3_$v -f python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c3_$v.log 2>&1
done

for L in tools/libfp8bs_head.so tools/libfp8bs_sched.so; do
  FP8BS_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grouped_schedule -c 3 python tools/grouped_c4_time.py 1 2>&1 | grep -E "duration" | tail -2
done
bash tools/ab_c4.sh tools/libfp8bs_head.so tools/libfp8bs_sched.so 3

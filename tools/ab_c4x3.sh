for i in 1 2 3; do
  for L in tools/libfp8bs_base.so tools/libfp8bs_ship.so tools/libfp8bs_pf.so; do echo -n "$L: "; FP8BS_LIB=$L timeout 300 python tools/grouped_c4_time.py 10 | sed 's/.*median/median/'; done
done

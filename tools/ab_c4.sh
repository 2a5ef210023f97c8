# same-box A/B of the C4 grouped Fprop: tools/ab_c4.sh libA libB [rounds]
R=${3:-3}
for i in $(seq 1 $R); do
  for L in "$1" "$2"; do echo -n "$L: "; FP8BS_LIB=$L timeout 300 python tools/grouped_c4_time.py 10; done
done

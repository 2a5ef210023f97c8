for i in 1 2; do for L in "$@"; do echo "$L"; FP8BS_LIB=$L timeout 300 python tools/quant_instep.py | grep -v again; done; done

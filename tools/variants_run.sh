# developer: time every build/variants/lib_*.so at the headline shape
for f in build/variants/lib_*.so; do echo "== $f"; TEMO_B200_LIB=$PWD/$f python tools/k1_check.py --no-hash --gens 3 --reps 5 "$@"; done

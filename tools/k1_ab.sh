# developer A/B: pair kernel vs generic kernel (checksums must match), then timings at the headline shape
for shape in "4096 5000 dtlz2" "1024 9000 dtlz3" "2048 512 dtlz2" "4096 5000 dtlz1" "1000 1280 dtlz4"; do set -- $shape
python tools/k1_check.py --pop $1 --dim $2 --problem $3 --gens 4 --reps 2
TEMO_B200_GENERIC_K1=1 python tools/k1_check.py --pop $1 --dim $2 --problem $3 --gens 4 --reps 2
done
TEMO_B200_K1_CAND_CAP=0 python tools/k1_check.py --pop 4096 --dim 5000 --gens 4 --reps 2
TEMO_B200_K1_CAND_CAP=1 python tools/k1_check.py --pop 4096 --dim 5000 --gens 4 --reps 2
python tools/k1_check.py --pop 4097 --dim 5000 --gens 3 --reps 2 --rng philox
TEMO_B200_GENERIC_K1=1 python tools/k1_check.py --pop 4097 --dim 5000 --gens 3 --reps 2 --rng philox
python tools/k1_check.py --no-hash --gens 3 --reps 5
TEMO_B200_K1_BOUND_ARRAYS=1 python tools/k1_check.py --pop 4096 --dim 5000 --gens 4 --reps 2

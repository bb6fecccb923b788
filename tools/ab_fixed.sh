# A/B of pass 1: fixed Cauchy-Schwarz reference (default) vs the exact running max,
# and the polynomial share of the exponentials for the fixed variant
for p in 8 10 12 14; do echo "fixed poly=$p"; PKV_POLY_PAIRS=$p python tools/time_score.py --iters 5; done
echo "exact poly=10"; PKV_SCORE_FIXED=0 python tools/time_score.py --iters 5

bash scripts/ab_time.sh cfg3 400 libtomo libtomo_pp libtomo_ppg

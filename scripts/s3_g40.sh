bash scripts/ab_time.sh cfg3 400 libtomo libtomo_h1 libtomo_h2 libtomo_h3

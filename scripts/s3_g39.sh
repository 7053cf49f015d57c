# ablations of the committed PCG kernel (timing only; results are wrong by construction)
bash scripts/ab_time.sh cfg3 400 libtomo libtomo_x0 libtomo_xc libtomo_xs libtomo_xq libtomo_xa

# group count at configs 5 and 4 (many small tile tasks per column at c5)
for g in 8 4 2 16; do FETI_SP_GROUPS=$g python scripts/factor_bench.py c5 3; done
for g in 4 16; do FETI_SP_GROUPS=$g python scripts/factor_bench.py c4 3; done

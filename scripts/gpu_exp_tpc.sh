# persistent tile-task kernel: tasks per CTA sweep (1 = one task per CTA, the round-1 launch shape)
for t in 1 2 3 4; do FETI_SP_TPC=$t python scripts/factor_bench.py c3; done
FETI_SP_TPC=2 python scripts/factor_bench.py c4 3
FETI_SP_TPC=1 python scripts/factor_bench.py c4 3

# factorization-schedule experiments (c3): group count, and potrf skipped
# (timing only: PO_SKIP_* leaves the factor wrong) -- how much of the
# factorization is the potrf chain
for g in 8 4 16; do FETI_SP_GROUPS=$g python scripts/factor_bench.py c3; done
python scripts/apply_bench.py c3; python scripts/apply_bench.py c4
FETI_NVCC_FLAGS="-DPO_SKIP_DIAG -DPO_SKIP_INV -DPO_SKIP_TRAIL -DPO_SKIP_PANEL" python -c "import sys; sys.path.insert(0,'.'); from paper_2502_08382_b200 import build; build.build(force=True)"
python scripts/factor_bench.py c3

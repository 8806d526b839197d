# potrf_invert_128 phase breakdown and shared-memory row stride (scripts/pb/*.bin built from potrf_bench.cu)
for b in base ld130 ld131 ld132 ld136 nodiag nopanel notrail noinv; do
  for nt in 8 148; do echo -n "$b "; ./scripts/pb/$b.bin $nt; done
done 2>&1 | tee gpurun_out/potrf_variants.txt

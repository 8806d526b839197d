# potrf_invert_128 before/after (scripts/pb/*.bin built from potrf_bench.cu against
# the header of a given commit): us per launch of NT tiles and the accuracy of L and inv(L)
for b in old new; do
  for nt in 8 148; do echo -n "$b "; ./scripts/pb/$b.bin $nt; done
done 2>&1 | tee gpurun_out/potrf_variants.txt

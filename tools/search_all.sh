{ echo "# Empirical top-k search on B200 (python -m paper_1305_1183_b200.cli search --top 4), round 1, after the block-contiguous stream kernel, bulk-store GEMVER stage 1 and the refreshed cost model (stream 1.09 / stream.dot 1.00 / tma.rank 0.99)."
echo "# Table-4 analogue (PAPER.md:572-602): rank-1 predicted combination vs best measured."
for spec in "GEMVER 32768 32768" "BICGK 16384 16384" "GESUMMV 32768 32768" "AXPYDOT 1 16777216" "VADD 1 268435456" "WAXPBY 1 268435456" "ATAX 16384 16384" "SGEMVT 16384 16384" "SGEMV 16384 16384" "MADD 16384 16384" "SSCAL 1 268435456"; do
  set -- $spec
  echo -n "$1 ${2}x${3}: "
  python -m paper_1305_1183_b200.cli search --sequence $1 --rows $2 --cols $3 --top 4 2>&1 | tail -1
done; } > gpurun_out/search2.txt 2>&1

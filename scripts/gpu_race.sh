set -x
timeout 1200 compute-sanitizer --tool racecheck --print-limit 5 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_racecheck2.log 2>&1
echo "racecheck exit $?"
grep -c "Race reported" gpurun_out/sanitize_racecheck2.log
grep -A3 "Race reported" gpurun_out/sanitize_racecheck2.log | head -8
python bench.py --steps 5 --warmup 3 --single-ordering --no-cpu-baseline --no-solve > gpurun_out/bench.json 2> gpurun_out/bench.log

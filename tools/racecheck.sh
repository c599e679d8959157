# racecheck with full hazard reports (run under gpurun): int path (C1, and C2
# with split-K units), float path (C3 at 4000 traces); -> gpurun_out/racecheck_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in "C1" "C2 2000 512" "C3 4000 0 0.02"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout -s KILL 900 $CS --tool racecheck --racecheck-report all --print-limit 40 python tools/repro.py $cfg \
      > gpurun_out/racecheck_$tag.log 2>&1
  echo "== $cfg: $(grep -E 'RACECHECK SUMMARY' gpurun_out/racecheck_$tag.log)"
done

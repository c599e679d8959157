mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool racecheck --racecheck-report all --print-limit 40 python tools/repro.py C1 > gpurun_out/racecheck_c1.log 2>&1
grep -v "^=========     \(Host\|#\|in \)" gpurun_out/racecheck_c1.log | head -120

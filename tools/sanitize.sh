# compute-sanitizer over the whole path (run under gpurun): int path (C1, and C2
# with split-K units) and float path (C3 at 4000 traces), class sums (C2-HW), and
# M >= 8192 int / float (the maxima-only finalize kernel); summary -> gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in "C1" "C2 2000 512" "C3 4000 0 0.02" "C2-HW 700" "C2 600 0 0 9002" "C3 600 0 0.02 8200"; do
    echo "== $tool $cfg" >> gpurun_out/sanitize.log
    CS_ENV=""; case "$cfg" in C2-HW*) CS_ENV="REPRO_CLASS_SUMS=1";; esac
    timeout -s KILL 900 env $CS_ENV $CS --tool $tool --error-exitcode 99 --print-limit 20 python tools/repro.py $cfg \
        > gpurun_out/san_tmp.log 2>&1
    echo "exit $?" >> gpurun_out/sanitize.log
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Invalid|Race|Barrier|Uninit)|key " gpurun_out/san_tmp.log | head -12 >> gpurun_out/sanitize.log
  done
done
cat gpurun_out/sanitize.log

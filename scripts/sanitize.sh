# compute-sanitizer over the hot kernels.
# memcheck (out-of-bounds / misaligned), racecheck (shared-memory hazards:
# K3's single-CTA hash rounds, K4's shared scans, K6/K7 staging), synccheck
# (barrier use), initcheck (uninitialised device reads).
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck; do
  for c in permute assign augment resize; do
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py $c \
      > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt

# compute-sanitizer over every libparse entry point (small calls) -> gpurun_out/san_<tool>.txt
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.txt 2>&1; echo "$t $?"
done

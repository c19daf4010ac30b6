#!/bin/bash
# Sweep LAMB_TUNE variants with short bench runs (no e2e/cpu); one JSON line each.
out=${1:-gpurun_out/sweep.jsonl}
: > $out
for t in "ua=4,ma=2,ub=4,mb=2" "ua=4,ma=3,ub=4,mb=3" "ua=4,ma=4,ub=4,mb=4" "ua=2,ma=3,ub=2,mb=3" "ua=2,ma=4,ub=2,mb=4"; do
  echo "{\"tune\": \"$t\"}" >> $out
  LAMB_TUNE=$t python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $out 2>&1
done

#!/bin/bash
# V-cycle time of the bench mapping for several configs (no profiler):
#   scripts/vc_times.sh C2/1 C3/1 C5/1   (extra env vars pass through)
for c in "$@"; do
  cfg=${c%/*}; sc=${c#*/}; [ "$sc" = "$c" ] && sc=1
  timeout 900 python scripts/vc_launches.py $cfg $sc 2>&1 | tail -1
done

#!/bin/bash
# Launch scripts/probes/tma_push_probe on n GPUs of this box (one process per GPU):
#   scripts/probes/tma_push_probe.sh <n> 
cd "$(dirname "$0")"
n=$1; 
idf=/tmp/ce_probe_id_$$
rm -f $idf
pids=""
for r in $(seq 0 $((n - 1))); do
  timeout 120 ./tma_push_probe $r $n $idf & pids="$pids $!"
done
rc=0
for p in $pids; do wait $p || rc=1; done
rm -f $idf
exit $rc

#!/bin/bash
# e2e (host buffers) sweep of the host pipeline chunk count for one config
cd "$(dirname "$0")/.."
C=${1:-c3}
for k in ${2:-3 4 5 6 8}; do
  ESN_PIPE_CHUNKS=$k timeout 300 python tools/e2e_probe.py $C 5 2>/dev/null | grep "e2e" | sed "s/^/chunks $k: /"
done

#!/bin/bash
# compute-sanitizer passes on a tiny fwd+bwd (GPU box). Usage: bash scripts/sanitize.sh
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool python scripts/tiny_fwd_bwd.py 2>&1 | grep -E "ERROR SUMMARY|ran|not supported|Error" | head -5
done

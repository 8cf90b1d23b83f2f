#!/bin/bash
# compute-sanitizer passes on small fwd+bwd+GEMM runs that hand several items to
# every persistent CTA (GPU box). Usage: bash scripts/sanitize.sh
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool python scripts/tiny_fwd_bwd.py > /tmp/san_$tool.txt 2>&1
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ran$|not supported" /tmp/san_$tool.txt | head -5
  # distinct reported race sites (racecheck), with counts
  grep -E "Race reported" /tmp/san_$tool.txt | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -10
done

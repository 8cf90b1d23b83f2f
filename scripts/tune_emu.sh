#!/bin/bash
# Build libhkattn with several forward exp-emulation fractions and probe each (GPU box).
for e128 in 2 3 4; do for e64 in 3 4 5; do
  HK_EXTRA="-DHK_FWD_EMU128=$e128 -DHK_FWD_EMU64=$e64" python -m paper_2511_08083_b200.build --force > /dev/null 2>&1 || { echo build failed; continue; }
  echo "emu128=$e128 emu64=$e64"; timeout 60 python scripts/probe.py --configs C2-nc,C3,C4-8192 --iters 10
done; done

#!/bin/bash
# Times every built kernel variant (paper_2605_25346_b200/libreach_b200_*.so) on the C4 sweep.
for so in paper_2605_25346_b200/libreach_b200_*.so; do
  case "$so" in *_phase.so) continue;; esac
  echo -n "$(basename $so): "
  REACH_B200_LIB=$so python tools/phase_profile.py 2>&1 | head -1
done

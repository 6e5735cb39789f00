#!/bin/bash
# Weight-stream ring sweep on the C4 sweep (product builds).
for lib in libreach_b200.so libreach_b200_w8.so; do
for cfg in "3 2048" "4 1536" "6 1024" "8 768" "4 2048" "6 2048" "5 2048"; do
  set -- $cfg
  echo -n "$lib RB_NSTAGE=$1 RB_STAGE_DOUBLES=$2: "
  RB_NSTAGE=$1 RB_STAGE_DOUBLES=$2 REACH_B200_LIB=paper_2605_25346_b200/$lib python tools/phase_profile.py 2>&1 | tail -1
done
done

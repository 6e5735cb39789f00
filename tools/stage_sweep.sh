#!/bin/bash
# Weight-stream ring sweep on the C4 sweep: product timing + phase breakdown.
for cfg in "3 2048" "4 2048" "6 1024" "8 1024" "4 1024" "8 512"; do
  set -- $cfg
  echo "== RB_NSTAGE=$1 RB_STAGE_DOUBLES=$2"
  RB_NSTAGE=$1 RB_STAGE_DOUBLES=$2 python tools/phase_profile.py 2>&1 | head -14
  RB_NSTAGE=$1 RB_STAGE_DOUBLES=$2 REACH_B200_LIB=paper_2605_25346_b200/libreach_b200.so python tools/phase_profile.py 2>&1 | head -1
done

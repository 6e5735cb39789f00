set -x
python tools/time_modes.py c4 fused,exact
REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_w10.so RB_NSTAGE=2 RB_STAGE_DOUBLES=4608 python tools/time_modes.py c4 fused,exact
REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_w10.so RB_NSTAGE=3 RB_STAGE_DOUBLES=3072 python tools/time_modes.py c4 fused
REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_w12.so RB_NSTAGE=2 RB_STAGE_DOUBLES=2688 python tools/time_modes.py c4 fused,exact
REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_w12.so RB_NSTAGE=3 RB_STAGE_DOUBLES=1792 python tools/time_modes.py c4 fused
REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_w12.so RB_NSTAGE=2 RB_STAGE_DOUBLES=2688 timeout 300 python -m pytest tests/test_gpu_dt.py -q -x

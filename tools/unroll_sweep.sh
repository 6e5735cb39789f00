# fused / exact C4 kernel time for row-loop unroll variants of the 12-warp DT kernel (built by hand into
# paper_2605_25346_b200/libreach_b200_<v>.so; see profiles/r02_c4_summary.md)
python tools/time_modes.py c4 fused,exact
for v in g2i4 g4i2 g8i4 g4i8; do echo "== $v"; REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_$v.so python tools/time_modes.py c4 fused,exact; done

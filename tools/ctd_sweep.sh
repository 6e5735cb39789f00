# ctl_reach_loss gradient at the C2 controller size for several persistent passes per SM
for s in 10 12 14; do RB_CTD_SLOTS_PER_SM=$s timeout 300 python tools/ctl_grad_bench.py 4 10; done
timeout 300 python -m pytest tests/test_gpu_ctl_grad.py tests/test_gpu_train.py -q

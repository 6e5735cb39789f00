for s in 0 4 8 16; do RB_CTD_SLOTS_PER_SM=$s timeout 300 python tools/ctl_grad_bench.py 4 10; done
RB_CTD_SLOTS_PER_SM=8 timeout 300 python -m pytest tests/test_gpu_ctl_grad.py -q

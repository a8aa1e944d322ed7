#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transfer_sep.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/chk2.log 2>&1; echo "rc $?" >> gpurun_out/chk2.log
STGMG_K1_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_k1_fgemm.py -x -q -p no:cacheprovider > gpurun_out/chk2p.log 2>&1; echo "rc $?" >> gpurun_out/chk2p.log
for c in 4 3 2; do timeout 400 python tools/kernel_times.py --config $c > gpurun_out/kt2_cfg$c.log 2>&1; done
for c in 4 3; do STGMG_K1_PERSIST=1 timeout 400 python tools/kernel_times.py --config $c > gpurun_out/kt2p_cfg$c.log 2>&1; done
timeout 300 python tools/lshape_table4.py --ref 2 --hf frozen > gpurun_out/t4f.log 2>&1
timeout 1000 python tools/lshape_table4.py --ref 3 --hf frozen >> gpurun_out/t4f.log 2>&1

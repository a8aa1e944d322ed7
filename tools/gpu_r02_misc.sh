#!/bin/bash
# separable restriction A/B + timings; Table 4 with the directional-face penalty h^-1 (hF mode 2)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_transfer_sep.py -x -q -p no:cacheprovider > gpurun_out/sep.log 2>&1; echo "rc $?" >> gpurun_out/sep.log
for c in 4 3 2; do timeout 400 python tools/kernel_times.py --config $c > gpurun_out/kts_cfg$c.log 2>&1; done
timeout 300 python tools/lshape_table4.py --ref 2 --hf dir_edge > gpurun_out/t4d.log 2>&1
timeout 1000 python tools/lshape_table4.py --ref 3 --hf dir_edge >> gpurun_out/t4d.log 2>&1

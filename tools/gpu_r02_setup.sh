#!/bin/bash
# Setup-time changes (GJ panel in shared memory with batched loads, zero-cell skip in the setup operator kernel):
# setup breakdown first (cheap), then the whole GPU suite.
mkdir -p gpurun_out
STGMG_SETUP_TIMES=1 timeout 300 python tools/setup_times.py 4 3 2 1 > gpurun_out/setup_s3b.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3b.log 2>&1; echo "rc $?" >> gpurun_out/pytest_s3b.log

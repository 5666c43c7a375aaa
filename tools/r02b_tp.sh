#!/bin/bash
O=gpurun_out/r02b_tp
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tp.py -q -x -rA > $O/pytest_tp.log 2>&1; tail -30 $O/pytest_tp.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log

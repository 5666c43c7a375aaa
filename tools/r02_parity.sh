#!/bin/bash
# round-2: parity at the benched configuration + the whole GPU suite
O=gpurun_out/r02_parity
mkdir -p $O
MK_PARITY_OUT=$O timeout 1500 python -m pytest tests/test_gpu_qwen3_8b.py -x -q -m gpu -rA > $O/pytest_qwen.log 2>&1; tail -15 $O/pytest_qwen.log
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_qwen3_8b.py > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log

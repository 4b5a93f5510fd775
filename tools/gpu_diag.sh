#!/usr/bin/env bash
# GPU parity tests + C2 diagnostics with the trace build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
BDSM_LIB=$PWD/paper_2401_17018_b200/libbdsm_b200_trace.so timeout 600 python tools/diag_c2.py --batches 8 ${DIAG_ARGS:-} > gpurun_out/diag.txt 2>&1
cat gpurun_out/diag.txt | grep -v "^  edge"

#!/bin/bash
# (compute-sanitizer is closed on the GPU pool this repo is measured on: runs left GPUs needing a reset;
# tests/test_gpu_configs.py::test_async_kernels_repeatable_and_exact is the stand-in.)
# compute-sanitizer over the TMA / mbarrier / tcgen05 kernels (scripts/sanitize_case.py), one tool
# per invocation: scripts/sanitize.sh racecheck|synccheck|memcheck  -> gpurun_out/sanitize_<tool>.txt
TOOL=${1:-racecheck}
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool "$TOOL" --print-limit 50 python scripts/sanitize_case.py \
    > gpurun_out/sanitize_${TOOL}.txt 2>&1
echo "exit $?" >> gpurun_out/sanitize_${TOOL}.txt
tail -5 gpurun_out/sanitize_${TOOL}.txt

#!/bin/bash
# Bounds-checked build (-DPXST_CHECKED: PXST_DCHECK device asserts in the
# splat, search and ring kernels) run over the GPU parity suite and the
# all-kernel workload.  compute-sanitizer is closed on this GPU pool, so this
# replaces memcheck; a failed check prints its condition and traps.
set -u
mkdir -p gpurun_out
export PXST_BUILD_DIR=build/checked PXST_LIB_OUT=paper_2003_12726_b200/libpxst_b200_checked.so
export PXST_NVCC_EXTRA="-DPXST_CHECKED"
python -c "import sys; sys.path.insert(0, '.'); from paper_2003_12726_b200 import build_native as b; b.build()"
export PXST_LIB=$PWD/paper_2003_12726_b200/libpxst_b200_checked.so
timeout 900 python tools/sanitize_workload.py > gpurun_out/checked_workload.log 2>&1
echo "workload rc=$?" > gpurun_out/checked_summary.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_spec.py \
  tests/test_gpu_loop.py tests/test_gpu_regularise.py -m gpu -q --timeout 900 > gpurun_out/checked_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/checked_summary.txt
tail -2 gpurun_out/checked_pytest.log >> gpurun_out/checked_summary.txt
grep -c "PXST_DCHECK failed" gpurun_out/checked_*.log >> gpurun_out/checked_summary.txt

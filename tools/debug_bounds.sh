#!/bin/bash
# Bounds-checked build (-DLX_DEBUG_BOUNDS: LX_DCHECK in the 3D two-step / slab kernels traps on an out-of-range
# plane, ring slot, piece, staging or ghost-delivery offset) run over the 3D and slab GPU tests.  A substitute
# for compute-sanitizer, which is closed on the GPU pool.  Run under gpurun from the repo root; the product
# library is rebuilt afterwards.
set -e
mkdir -p gpurun_out
NVCC_EXTRA="-DLX_DEBUG_BOUNDS" python -c "from paper_2310_08344_b200 import _build; _build.build(force=True)"
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_parity.py -q -k "3d or 3D or slab" \
    > gpurun_out/debug_bounds.log 2>&1 || echo "pytest rc $?" >> gpurun_out/debug_bounds.log
tail -3 gpurun_out/debug_bounds.log
python -c "from paper_2310_08344_b200 import _build; _build.build(force=True)"

#!/usr/bin/env bash
# A/B: staged keyframe uploads waited for by the kernels (device flags written
# by the copy stream) vs stream event waits; full GPU tests first; then the
# clean e2e diagnostic and the 8-step bench with e2e, per library.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/abf2_tests.log
cat gpurun_out/abf2_tests.log
for r in 1 2; do
for tag in base flags; do
  RF_LIB_PATH=$PWD/variants/lib_$tag.so KF=400 timeout 900 python tools/diag_e2e_profile.py 2>/dev/null | head -2 | sed "s/^/$tag /"
done; done

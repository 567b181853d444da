#!/bin/bash
# programmatic dependent launch for the TMA, pair and multi-step kernels: full GPU suite, A/B
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r2aq.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/gputest_r2aq.log
for v in base pdl base pdl; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 20; HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base pdl; do HFTW_LIBRARY=tools/exp/$v.so python tools/stencil_multi.py 100 | tail -1; HFTW_LIBRARY=tools/exp/$v.so timeout 600 python tools/group_one_gpu.py 40 2x4 | tail -1; done

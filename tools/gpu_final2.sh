#!/bin/bash
# final round-2 evidence: smoke, full GPU suite, then the evidence set of gpu_r2s.sh
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final2.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/gputest_final2.log
bash tools/gpu_r2s.sh r02h2

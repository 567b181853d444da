#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r2ad.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputest_r2ad.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

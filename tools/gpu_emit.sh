#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_emit_gpu.py tests/test_cpp_adapter.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -15

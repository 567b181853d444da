#!/bin/bash
# multi-sweep diffusion on 256x256x64: wave chunk height and strip width (tuning build)
cd $GRAFT_REPO_ROOT
for c in 8 6 4 2 12; do echo "chunk $c: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_WAVE_CHUNK=$c python tools/stencil_multi.py 100 | grep multi | tail -1)"; done
for c in 8 4; do echo "tx32 chunk $c: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_TX=32 HFTW_WAVE_CHUNK=$c python tools/stencil_multi.py 100 | tail -2 | tr '\n' ' ')"; done

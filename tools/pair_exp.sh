# timing experiments on the pair kernel: build variants with -D flags and time each
set -e
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --fmad=false -Xcompiler -fPIC,-ffp-contract=off -shared -cudart static"
for v in "$@"; do
  mkdir -p /tmp/exp_$v
  $NV -D$v -o /tmp/exp_$v/libhftw.so paper_1802_05839_b200/csrc/hftw.cu
done

// PCIe probe: device->host by the copy engine (cudaMemcpyAsync) vs by SM stores into
// mapped pinned host memory (zero-copy), alone and next to a copy-engine H2D stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zerocopy_probe tools/zerocopy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void store_to_host(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = (size_t)1 << 30, n2 = bytes / 16;
    double *dsrc, *ddst, *h1, *h2;
    cudaMalloc(&dsrc, bytes);
    cudaMalloc(&ddst, bytes);
    cudaMemset(dsrc, 1, bytes);
    cudaHostAlloc(&h1, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
    double2* hdev = nullptr;
    cudaHostGetDevicePointer((void**)&hdev, h1, 0);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto timed = [&](auto fn, const char* name, double gb) {
        for (int r = 0; r < 2; ++r) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, 0);
            fn();
            cudaDeviceSynchronize();
            cudaEventRecord(b, 0);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (r == 1) printf("%-48s %7.1f GB/s (%.1f ms)\n", name, gb / (ms * 1e-3), ms);
        }
    };
    const double gb = bytes / 1e9;
    timed([&] { cudaMemcpyAsync(h1, dsrc, bytes, cudaMemcpyDeviceToHost, s1); }, "D2H copy engine", gb);
    for (int blocks : {sms, 2 * sms, 4 * sms, 8 * sms}) {
        char nm[64];
        snprintf(nm, sizeof nm, "D2H SM stores, %d blocks", blocks);
        timed([&] { store_to_host<<<blocks, 512, 0, s1>>>((const double2*)dsrc, hdev, n2); }, nm, gb);
    }
    timed([&] {
        cudaMemcpyAsync(h1, dsrc, bytes, cudaMemcpyDeviceToHost, s1);
        cudaMemcpyAsync(ddst, h2, bytes, cudaMemcpyHostToDevice, s2);
    }, "D2H CE + H2D CE (D2H-equivalent of both)", gb);
    timed([&] {
        store_to_host<<<2 * sms, 512, 0, s1>>>((const double2*)dsrc, hdev, n2);
        cudaMemcpyAsync(ddst, h2, bytes, cudaMemcpyHostToDevice, s2);
    }, "D2H SM stores + H2D CE (per direction)", gb);
    timed([&] {
        cudaMemcpyAsync(h1, dsrc, bytes / 2, cudaMemcpyDeviceToHost, s1);
        store_to_host<<<2 * sms, 512, 0, s2>>>((const double2*)(dsrc) + n2 / 2, hdev + n2 / 2, n2 / 2);
    }, "D2H half CE + half SM stores", gb);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// tools/tma_probe.cu -- probes which tensor-map shapes the B200 TMA accepts.
// usage: tma_probe <rank 2|3> <box0> <box1> <box2> <l2promo 0..3> <c0> [<dim0>]
//   fp64 tensor {dim0 (default 64), 20, 8}; prints whether the load faults.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int nbytes, int c0, int c1, int c2) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(nbytes) : "memory");
        if (RANK == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(smem)), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(smem)), "l"(&tm), "r"(c0), "r"(c1), "r"(su32(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)) : "memory");
        out[0] = ((double*)smem)[0];
        out[1] = ((double*)smem)[1];
    }
}

int main(int argc, char** argv) {
    int rank = atoi(argv[1]), b0 = atoi(argv[2]), b1 = atoi(argv[3]), b2 = atoi(argv[4]);
    int promo = atoi(argv[5]), c0 = atoi(argv[6]);
    long long P = argc > 7 ? atoll(argv[7]) : 64, R = 20, Z = 8;
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    double* buf;
    cudaMalloc(&buf, P * R * Z * 8);
    double* h = (double*)malloc(P * R * Z * 8);
    for (long long i = 0; i < P * R * Z; ++i) h[i] = (double)i;
    cudaMemcpy(buf, h, P * R * Z * 8, cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, 4096);
    CUtensorMap tm;
    cuuint32_t es[3] = {1, 1, 1};
    cuuint64_t dims[3] = {(cuuint64_t)P, (cuuint64_t)R, (cuuint64_t)Z};
    cuuint64_t str[2] = {(cuuint64_t)P * 8, (cuuint64_t)P * R * 8};
    cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, buf, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int nbytes = b0 * b1 * (rank == 3 ? b2 : 1) * 8;
    int smem = 200000;
    cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (rank == 3) k<3><<<1, 32, smem>>>(tm, out, nbytes, c0, 2, 0);
    else k<2><<<1, 32, smem>>>(tm, out, nbytes, c0, 2, 0);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[2] = {-1, -1};
    cudaMemcpy(ho, out, 16, cudaMemcpyDeviceToHost);
    printf("rank %d box {%d,%d,%d} promo %d c0 %d dim0 %lld: encode=%d %s out=%g %g (expect %g)\n", rank, b0, b1,
           b2, promo, c0, P, (int)r, cudaGetErrorString(e), ho[0], ho[1], (double)(2 * P + c0));
    return e != cudaSuccess;
}

// Minimal TMA + mbarrier check mirroring relax_tiled.cu's usage (diagnostic).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_1703_07206_b200/csrc/device.cuh"
using namespace sgmlb;

struct __align__(128) Sm {
    double u[2][352];
    double g[2][256];
    unsigned long long full[2];
};

__global__ void k(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tg, double* out,
                  int c0, int c1, int c2, int use_tma) {
    extern __shared__ __align__(128) unsigned char raw[];
    Sm& S = *reinterpret_cast<Sm*>(raw);
    if (threadIdx.x == 0) {
        mbar_init(&S.full[0], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&S.full[0], 34 * 10 * 8 + (use_tma == 2 ? 32 * 8 * 8 : 0));
        if (use_tma) tma_load_3d(S.u[0], &tm, c0, c1, c2, &S.full[0]);
        if (use_tma == 2) tma_load_3d(S.g[0], &tg, c0, c1, c2, &S.full[0]);
    }
    if (use_tma) mbar_wait(&S.full[0], 0);
    __syncthreads();
    for (int e = threadIdx.x; e < 340; e += blockDim.x) out[e] = S.u[0][e];
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 17, Ne = N + 2, Px = (Ne + 1) / 2 * 2;
    const size_t n = (size_t)Px * Ne * Ne;
    double* h = new double[n];
    for (size_t i = 0; i < n; ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 340 * 8);
    cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)Ne, (cuuint64_t)Ne, (cuuint64_t)Ne};
    cuuint64_t str[2] = {(cuuint64_t)Px * 8, (cuuint64_t)Px * Ne * 8};
    cuuint32_t box[3] = {34, 10, 1}, es[3] = {1, 1, 1};
    CUtensorMap mg;
    cuuint32_t boxg[3] = {32, 8, 1};
    CUresult rcg = enc(&mg, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode g rc=%d\n", (int)rcg);
    CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d (box 34 > Ne=%d)\n", (int)rc, Ne);
    for (int use : {0, 1, 2}) {
        int cx = argc > 2 ? atoi(argv[2]) : 0, cy = argc > 3 ? atoi(argv[3]) : 0;
        k<<<1, 128, sizeof(Sm)>>>(m, mg, o, cx, cy, 1, use);
        cudaError_t e = cudaDeviceSynchronize();
        printf("use_tma=%d -> %s\n", use, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    double r[340];
    cudaMemcpy(r, o, 340 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 10; ++y)
        for (int x = 0; x < 34; ++x) {
            double want = (x < Ne && y < Ne) ? (double)(x + (size_t)Px * (y + (size_t)Ne * 1)) : 0.0;
            if (r[y * 34 + x] != want) ++bad;
        }
    printf("mismatches %d\n", bad);
    return 0;
}

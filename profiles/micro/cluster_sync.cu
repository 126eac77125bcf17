// Micro-benchmark: cost of a cluster barrier round on B200 (cluster of 8, 256 threads), bare and with
// DSMEM stores / loads before it. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) k_sync(int iters, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double buf[2][512];
    const int q = int(cl.block_rank());
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        if (MODE == 1) {  // every warp's lanes 0..7 store one double into each CTA (like the p push)
            if ((threadIdx.x & 31) < 8) cl.map_shared_rank(&buf[par][0], threadIdx.x & 31)[(threadIdx.x >> 5) + 8 * q] = it;
        }
        if (MODE == 2) {  // remote loads of 343 values
            for (int i = threadIdx.x; i < 343; i += blockDim.x) acc += cl.map_shared_rank(&buf[par][0], i % 8)[i];
        }
        if (MODE == 3) __syncthreads();
        if (MODE != 3) cl.sync();
        if (MODE == 1) acc += buf[par][threadIdx.x & 63];
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 3410;
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k_sync<0><<<8, 256>>>(iters, out);
            if (mode == 1) k_sync<1><<<8, 256>>>(iters, out);
            if (mode == 2) k_sync<2><<<8, 256>>>(iters, out);
            if (mode == 3) k_sync<3><<<8, 256>>>(iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("mode %d (%s): %.3f us per round\n", mode,
                            mode == 0 ? "cluster.sync" : mode == 1 ? "DSMEM stores + cluster.sync"
                                                   : mode == 2 ? "DSMEM loads + cluster.sync" : "__syncthreads",
                            1e3 * ms / iters);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// NVLink exchange ceilings on a B200 pair (one process, two devices, peer
// access): copy engine, SM pull (remote loads), SM push (remote stores) and
// TMA bulk pull at several request sizes; one and both directions at once.
// Standalone probe for the exchange design (profiles/r2_nvlink_modes.txt):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvm scripts/nvlink_modes.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * st < n16; i += 4 * st) {
        uint4 a = src[i], b = src[i + st], c = src[i + 2 * st], d = src[i + 3 * st];
        dst[i] = a; dst[i + st] = b; dst[i + 2 * st] = c; dst[i + 3 * st] = d;
    }
    for (; i < n16; i += st) dst[i] = src[i];
}

// TMA bulk pull: each CTA copies `req` bytes per request into smem (2 stages),
// then streams them to dst with 16-byte stores.
__global__ void k_bulk(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t bytes,
                       uint32_t req) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar[2];
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&mbar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t nreq = bytes / req;
    uint32_t ph[2] = {0, 0};
    size_t r = blockIdx.x;
    auto issue = [&](size_t rr, int s) {
        if (tid == 0 && rr < nreq) {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(req) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * req)), "l"(src + rr * req), "r"(req), "r"(mb) : "memory");
        }
    };
    issue(r, 0);
    int s = 0;
    for (; r < nreq; r += gridDim.x) {
        issue(r + gridDim.x, s ^ 1);
        const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(mb), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
        const uint4* a = reinterpret_cast<const uint4*>(sm + s * req);
        uint4* d = reinterpret_cast<uint4*>(dst + r * req);
        for (uint32_t j = tid; j < req / 16; j += blockDim.x) d[j] = a[j];
        __syncthreads();
        s ^= 1;
    }
}

int main() {
    const size_t bytes = 256ull << 20;
    uint8_t *b[2][2];  // [dev][0 = src, 1 = dst]
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&b[d][0], bytes));
        CK(cudaMalloc(&b[d][1], bytes));
        CK(cudaMemset(b[d][0], d + 1, bytes));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 49152));
    }
    // mode: 0 CE pull, 1 SM pull, 2 SM push, 3.. TMA pull with request sizes
    const uint32_t reqs[] = {672, 2048, 8192, 24576, 49152};
    const char* names[] = {"copy engine (cudaMemcpyPeerAsync)", "SM pull (remote 16B loads)",
                           "SM push (remote 16B stores)"};
    for (int mode = 0; mode < 3 + 5; ++mode) {
        for (int both = 0; both < 2; ++both) {
            float best = 1e9f;
            for (int rep = 0; rep < 8; ++rep) {
                for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
                for (int d = 0; d < (both ? 2 : 1); ++d) {
                    CK(cudaSetDevice(d));
                    const int p = 1 - d;
                    CK(cudaEventRecord(e0[d], st[d]));
                    if (mode == 0) {
                        CK(cudaMemcpyPeerAsync(b[d][1], d, b[p][0], p, bytes, st[d]));
                    } else if (mode == 1) {
                        k_copy<<<148 * 4, 512, 0, st[d]>>>((const uint4*)b[p][0], (uint4*)b[d][1], bytes / 16);
                    } else if (mode == 2) {
                        k_copy<<<148 * 4, 512, 0, st[d]>>>((const uint4*)b[d][0], (uint4*)b[p][1], bytes / 16);
                    } else {
                        const uint32_t rq = reqs[mode - 3];
                        const int per_sm = rq <= 8192 ? 4 : 2;
                        k_bulk<<<148 * per_sm, 256, 2 * rq, st[d]>>>(b[p][0], b[d][1], bytes - bytes % rq, rq);
                    }
                    CK(cudaEventRecord(e1[d], st[d]));
                }
                float worst = 0.f;  // both directions: the slower one
                for (int d = 0; d < (both ? 2 : 1); ++d) {
                    CK(cudaSetDevice(d));
                    CK(cudaEventSynchronize(e1[d]));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
                    worst = ms > worst ? ms : worst;
                }
                if (rep > 1 && worst < best) best = worst;
            }
            char nm[64];
            if (mode >= 3) snprintf(nm, sizeof nm, "TMA bulk pull, %u-byte requests", reqs[mode - 3]);
            printf("%-40s %-13s %8.1f GB/s per direction\n", mode < 3 ? names[mode] : nm,
                   both ? "bidirectional" : "one way", bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}

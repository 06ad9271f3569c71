// NCCL send/recv between two B200s (one process, ncclCommInitAll): plain
// cudaMalloc buffers vs ncclMemAlloc buffers registered with
// ncclCommRegister (user-buffer registration: NVLink P2P may then copy
// straight between the user buffers instead of through NCCL's FIFO).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/nccl_reg_probe.bin \
//        scripts/nccl_reg_probe.cu -lnccl
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)
#define NK(x) do { ncclResult_t r = (x); if (r != ncclSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, ncclGetErrorString(r)); exit(1); } } while (0)

int main() {
    int ver = 0;
    NK(ncclGetVersion(&ver));
    printf("nccl %d\n", ver);
    ncclComm_t comm[2];
    int devs[2] = {0, 1};
    NK(ncclCommInitAll(comm, 2, devs));
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
    }
    const size_t sizes[] = {10ull << 20, 40ull << 20, 80ull << 20, 160ull << 20};
    for (int reg = 0; reg < 2; ++reg) {
        void *sb[2], *rb[2], *hs[2] = {nullptr, nullptr}, *hr[2] = {nullptr, nullptr};
        const size_t cap = 160ull << 20;
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            if (reg) {
                NK(ncclMemAlloc(&sb[d], cap));
                NK(ncclMemAlloc(&rb[d], cap));
                NK(ncclCommRegister(comm[d], sb[d], cap, &hs[d]));
                NK(ncclCommRegister(comm[d], rb[d], cap, &hr[d]));
            } else {
                CK(cudaMalloc(&sb[d], cap));
                CK(cudaMalloc(&rb[d], cap));
            }
            CK(cudaMemset(sb[d], d + 1, cap));
        }
        for (size_t bytes : sizes) {
            float best = 1e9f;
            for (int rep = 0; rep < 12; ++rep) {
                for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
                for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
                NK(ncclGroupStart());
                for (int d = 0; d < 2; ++d) {
                    NK(ncclSend(sb[d], bytes, ncclUint8, 1 - d, comm[d], st[d]));
                    NK(ncclRecv(rb[d], bytes, ncclUint8, 1 - d, comm[d], st[d]));
                }
                NK(ncclGroupEnd());
                float worst = 0.f;
                for (int d = 0; d < 2; ++d) {
                    CK(cudaSetDevice(d));
                    CK(cudaEventRecord(e1[d], st[d]));
                    CK(cudaEventSynchronize(e1[d]));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
                    worst = ms > worst ? ms : worst;
                }
                if (rep > 2 && worst < best) best = worst;
            }
            printf("%-34s %4zu MB  %7.3f ms  %7.1f GB/s received per GPU\n",
                   reg ? "ncclMemAlloc + ncclCommRegister" : "cudaMalloc", bytes >> 20, best,
                   bytes / (best * 1e-3) / 1e9);
        }
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            if (reg) {
                NK(ncclCommDeregister(comm[d], hs[d]));
                NK(ncclCommDeregister(comm[d], hr[d]));
                NK(ncclMemFree(sb[d]));
                NK(ncclMemFree(rb[d]));
            } else {
                CK(cudaFree(sb[d]));
                CK(cudaFree(rb[d]));
            }
        }
    }
    for (int d = 0; d < 2; ++d) ncclCommDestroy(comm[d]);
    return 0;
}

// HBM streaming probe (diagnostic, not part of libbass): every CTA streams
// `per_cta` bytes of a large buffer into a ring of `stages` 16 KB shared-
// memory slots with 1-D bulk copies (cp.async.bulk + mbarrier), consuming
// nothing — the weight-stream skeleton of the GEMMs.  Reports achieved GB/s
// for (grid, stages, bytes per CTA), which tells how much data must be in
// flight per SM to saturate HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const char* __restrict__ src, long long per_cta, int stages, long long total) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + stages * 16384);
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long n = per_cta / 16384;
    const char* base = src + ((long long)blockIdx.x * per_cta) % total;
    for (long long i = 0; i < n + stages; ++i) {
        if (i >= stages) {   // wait for the copy issued `stages` iterations ago
            const int s = (int)((i - stages) % stages);
            const uint32_t par = (uint32_t)(((i - stages) / stages) & 1);
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                    : "=r"(ok)
                    : "r"(su32(&bars[s])), "r"(par)
                    : "memory");
        }
        if (i < n) {
            const int s = (int)(i % stages);
            const uint32_t bar = su32(&bars[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(bar) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                             su32(sm + s * 16384)),
                         "l"(base + i * 16384), "r"(bar)
                         : "memory");
        }
    }
}

int main() {
    const long long total = 4ll << 30;   // 4 GiB >> L2
    char* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384 + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grids[] = {sms / 2, sms, 2 * sms};
    const int stages_list[] = {1, 2, 3, 4, 6, 8, 12};
    const long long per[] = {256 << 10, 1 << 20, 4 << 20};
    for (int g : grids)
        for (int st : stages_list)
            for (long long p : per) {
                const size_t smem = st * 16384 + 1024;
                if (g > sms && smem > 110 * 1024) continue;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    probe<<<g, 32, smem>>>(buf, p, st, total);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                }
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = (double)g * p / (ms / 1e3) / 1e9;
                printf("{\"grid\": %d, \"stages\": %d, \"per_cta_kb\": %lld, \"us\": %.2f, \"GB/s\": %.1f, \"GB/s_per_cta\": %.1f}\n",
                       g, st, p >> 10, ms * 1e3, gbs, gbs / g);
            }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}

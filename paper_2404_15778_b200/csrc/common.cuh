// Shared device helpers for libbass (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#define BASS_DEV __device__ __forceinline__

namespace bass {

constexpr int kWarp = 32;

// Programmatic dependent launch: allow the next (PDL-launched) kernel in the
// stream to start its prologue now; it still waits (griddepcontrol.wait) for
// this grid's completion before touching our outputs.
BASS_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Wait until the preceding kernel in the stream has completed and its writes
// are visible (no-op when the kernel was not launched with PDL).  Every
// PDL-launched kernel calls this before its first dependent global access.
BASS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Per-CTA timeline trace (diagnostics): when buf != nullptr, CTA i of a traced
// launch writes {t_start, t_end, smid, tag} (globaltimer ns) at record base + i.
struct TraceArg {
    unsigned long long* buf;
    long long base;
    int tag;
};
BASS_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
BASS_DEV void trace_end(const TraceArg& tr, unsigned long long t0) {
    if (tr.buf && threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        unsigned long long* r = tr.buf + 4 * (tr.base + blockIdx.x);
        r[0] = t0;
        r[1] = gtimer();
        r[2] = sm;
        r[3] = (unsigned long long)tr.tag;
    }
}

// cudaFuncSetAttribute is per device: run `f` once per (call site, device).
// `mask` is the call site's static bit set of devices already configured.
template <typename F>
inline void once_per_device(unsigned& mask, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = 1u << (dev & 31);
    if (!(mask & bit)) {
        f();
        mask |= bit;
    }
}

// Launch with programmatic stream serialization (PDL).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Packed weight layout for the tcgen05 GEMM: [N, K] output-major matrices are
// stored as 128 x 64 tiles (16 KB each), tile (nt, kb) at ((nt * K/64) + kb),
// each tile the exact shared-memory image of a K-major 128-byte-swizzled UMMA
// operand (row r at r * 128 B, 16-byte chunk c at (c ^ (r & 7)) * 16 B).  A
// CTA's weight stream is then a run of contiguous 16 KB blocks (1-D bulk
// copies, full DRAM pages) instead of 128-byte row pieces.
BASS_DEV int64_t packed_index(int64_t n, int64_t k, int64_t K) {
    const int64_t tile = (n >> 7) * (K >> 6) + (k >> 6);
    const int r = (int)(n & 127), c = (int)((k & 63) >> 3);
    return tile * 8192 + r * 64 + ((c ^ (r & 7)) << 3) + (k & 7);
}
inline int64_t packed_rows(int64_t N) { return (N + 127) / 128 * 128; }

// element access in either storage dtype; all math is fp32 (or fp64 for sampling)
BASS_DEV float ld(const float* p, int64_t i) { return p[i]; }
BASS_DEV float ld(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
BASS_DEV void st(float* p, int64_t i, float v) { p[i] = v; }
BASS_DEV void st(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

template <typename T> BASS_DEV T cvt(float v);
template <> BASS_DEV float cvt<float>(float v) { return v; }
template <> BASS_DEV __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

BASS_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
BASS_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
BASS_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// orderable key of a float: larger float -> larger key (NaN-free input)
BASS_DEV uint32_t fkey(float x) {
    uint32_t u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// (value, index) argmax with first-index tie break (np.argmax semantics)
struct ArgMax {
    float v;
    int i;
};
BASS_DEV ArgMax better(ArgMax a, ArgMax b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}
BASS_DEV ArgMax warp_argmax(ArgMax a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax b{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.i, o)};
        a = better(a, b);
    }
    return a;
}

// Deterministic block reductions (fixed tree; identical result every launch).
// `scratch` must hold blockDim.x/32 elements.
template <typename T>
BASS_DEV T block_sum(T v, T* scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    T r = 0;
    if (w == 0) {
        r = lane < nw ? scratch[lane] : T(0);
        r = warp_sum(r);
        if (lane == 0) scratch[0] = r;
    }
    __syncthreads();
    r = scratch[0];
    __syncthreads();
    return r;
}

BASS_DEV float block_max(float v, float* scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        float r = lane < nw ? scratch[lane] : -INFINITY;
        r = warp_max(r);
        if (lane == 0) scratch[0] = r;
    }
    __syncthreads();
    float r = scratch[0];
    __syncthreads();
    return r;
}

BASS_DEV ArgMax block_argmax(ArgMax a, float* sv, int* si) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    a = warp_argmax(a);
    __syncthreads();
    if (lane == 0) { sv[w] = a.v; si[w] = a.i; }
    __syncthreads();
    if (w == 0) {
        ArgMax r{-INFINITY, 0x7fffffff};
        if (lane < nw) r = ArgMax{sv[lane], si[lane]};
        r = warp_argmax(r);
        if (lane == 0) { sv[0] = r.v; si[0] = r.i; }
    }
    __syncthreads();
    ArgMax r{sv[0], si[0]};
    __syncthreads();
    return r;
}

// Exclusive block scan of one value per thread (fixed order).  `scratch`
// holds 33 elements.  Returns the exclusive prefix; *total = sum.
// Not inlined: inlined into the sampled-verify kernel, nvcc 12.9 derived the
// warp slot of `scratch[w]` as (tid >> 3) without the low-bit mask — a
// misaligned shared store (compute-sanitizer, C3 sampled config).
template <typename T>
__device__ __noinline__ T block_exclusive_scan(T v, T* scratch, T* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    T excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = T(0);
    __syncthreads();
    if (lane == 31) scratch[w] = incl;
    __syncthreads();
    if (w == 0) {
        T s = lane < nw ? scratch[lane] : T(0);
        T si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T n = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += n;
        }
        T se = __shfl_up_sync(0xffffffffu, si, 1);
        if (lane == 0) se = T(0);
        if (lane < nw) scratch[lane] = se;       // exclusive warp offsets
        if (lane == nw - 1) scratch[32] = si;    // total
    }
    __syncthreads();
    T off = scratch[w];
    T tot = scratch[32];
    __syncthreads();
    *total = tot;
    return off + excl;
}

}  // namespace bass

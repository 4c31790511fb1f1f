// common.cuh -- device helpers shared by the WildCat sm_100a kernels.
// (Product path only; the fp64 CPU oracle under oracle/ shares nothing with this.)
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace wc {

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels of a stream-ordered chain are launched with programmatic stream serialisation, so the
// launch of kernel N+1 overlaps the tail of kernel N; every such kernel calls pdl_wait() before it
// touches anything kernel N wrote (griddepcontrol.wait returns at once when launched normally).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kWarp = 32;

// ---------------------------------------------------------------- element loads
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ double to_f64(float x) { return (double)x; }
__device__ __forceinline__ double to_f64(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// Load 8 consecutive elements (16- or 32-byte aligned) and widen to fp64 (exact).
template <typename T> struct Vec8;
template <> struct Vec8<__nv_bfloat16> {
    static __device__ __forceinline__ void load(const __nv_bfloat16 *p, double out[8]) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            out[2 * k] = (double)__uint_as_float(wd[k] << 16);
            out[2 * k + 1] = (double)__uint_as_float(wd[k] & 0xffff0000u);
        }
    }
};
template <> struct Vec8<float> {
    static __device__ __forceinline__ void load(const float *p, double out[8]) {
        const float4 x = __ldg(reinterpret_cast<const float4 *>(p));
        const float4 y = __ldg(reinterpret_cast<const float4 *>(p) + 1);
        out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
        out[4] = y.x; out[5] = y.y; out[6] = y.z; out[7] = y.w;
    }
};

// 8 consecutive raw elements kept as 16-byte vectors (bf16: one, fp32: two) until they are used;
// at(k) widens element k exactly to fp64.
template <typename T> struct Raw8;
template <> struct Raw8<__nv_bfloat16> {
    uint4 v;
    __device__ __forceinline__ void load(const __nv_bfloat16 *p) { v = __ldg(reinterpret_cast<const uint4 *>(p)); }
    __device__ __forceinline__ double at(int k) const {
        const uint32_t wd = k < 2 ? v.x : k < 4 ? v.y : k < 6 ? v.z : v.w;
        return (double)__uint_as_float((k & 1) ? (wd & 0xffff0000u) : (wd << 16));
    }
};
template <> struct Raw8<float> {
    float4 a, b;
    __device__ __forceinline__ void load(const float *p) {
        a = __ldg(reinterpret_cast<const float4 *>(p));
        b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    }
    __device__ __forceinline__ double at(int k) const {
        const float4 &q = k < 4 ? a : b;
        const int kk = k & 3;
        return (double)(kk == 0 ? q.x : kk == 1 ? q.y : kk == 2 ? q.z : q.w);
    }
};

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based generator of Salmon et al. (SC'11).  The pivot uniform of round i of
// unit u is built from Philox4x32-10(key = seed, ctr = (i, u_lo, u_hi, 'PIVT')) with
// 53 random bits (reading Z2).
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int rnd = 0; rnd < 10; ++rnd) {
        const uint32_t lo0 = 0xD2511F53u * c[0];
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0;
        const uint32_t n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__device__ __forceinline__ double pivot_uniform(uint64_t seed, uint32_t round_i, uint64_t unit) {
    uint32_t c[4] = {round_i, (uint32_t)unit, (uint32_t)(unit >> 32), 0x50495654u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double a = (double)(c[0] >> 5), b = (double)(c[1] >> 6);
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------- Lambert W0 (device)
// Loczi iteration, 6 steps; z >= e uses log z - log log z.
__device__ __forceinline__ double lambert_w0_dev(double z) {
    if (z == 0.0) return 0.0;
    const double lz = log(z);
    double b = (z >= 2.718281828459045) ? lz - log(lz) : exp(lz - 1.0);
#pragma unroll
    for (int k = 0; k < 6; ++k) b = b / (1.0 + b) * (1.0 + lz - log(b));
    return b;
}

// ---------------------------------------------------------------- reductions
// Warp index computed through opaque PTX.  With a plain `threadIdx.x >> 5`, nvcc 12.9 (sm_100a)
// folded `&scratch[w]` into `scratch_bytes + (tid >> 2)` -- correct only for lanes 0..3 -- and
// reused it for every lane (misaligned shared access).  The opaque shift blocks that rewrite.
__device__ __forceinline__ int warp_index() {
    int w;
    asm volatile("shr.u32 %0, %1, 5;" : "=r"(w) : "r"((unsigned)threadIdx.x));
    return w;
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T> __device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum (fixed tree order); result valid in all threads.
// `scratch` needs blockDim/32 doubles.  Contains __syncthreads.
__device__ __forceinline__ double block_sum(double v, double *scratch) {
    const int lane = threadIdx.x & 31, w = warp_index(), nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = lane < nw ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    t = scratch[0];
    __syncthreads();
    return t;
}

__device__ __forceinline__ double block_max(double v, double *scratch) {
    const int lane = threadIdx.x & 31, w = warp_index(), nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        double t = lane < nw ? scratch[lane] : -1.0e308;
        t = warp_max(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    const double t = scratch[0];
    __syncthreads();
    return t;
}

// Block-wide exclusive scan of one double per thread in a fixed order (warp shuffle
// scan + scan of warp totals).  Returns the exclusive prefix; *total gets the sum.
__device__ __forceinline__ double block_exclusive_scan(double v, double *scratch, double *total) {
    const int lane = threadIdx.x & 31, w = warp_index(), nw = blockDim.x >> 5;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const double wtot = __shfl_sync(0xffffffffu, incl, 31);
    __syncthreads();
    if (lane == 0) scratch[w] = wtot;
    __syncthreads();
    if (w == 0) {
        double t = lane < nw ? scratch[lane] : 0.0;
        double ti = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) ti += y;
        }
        if (lane < nw) scratch[lane] = ti - t;  // exclusive warp offsets
        if (lane == nw - 1) scratch[32] = ti;
    }
    __syncthreads();
    const double excl = scratch[w] + (incl - v);
    *total = scratch[32];
    __syncthreads();
    return excl;
}

// ---------------------------------------------------------------- grid-group barrier
// Barrier among the `count` co-resident CTAs that share `ctr` (one counter per unit).
// Monotone counter: the e-th barrier waits until ctr >= e*count.  The caller zeroes
// ctr before the launch.  Release/acquire at gpu scope orders the global writes.
__device__ __forceinline__ void group_barrier(unsigned int *ctr, unsigned int count, unsigned int epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
        const unsigned int target = epoch * count;
        unsigned int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// ---------------------------------------------------------------- mbarrier + bulk async copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar` in bytes.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// L2 eviction-priority policies (createpolicy) and cache-hinted bulk copy / store.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void st_f64_hint(double *p, double v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(policy) : "memory");
}
__device__ __forceinline__ void st_f64x2_hint(double *p, double a, double b, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(policy)
                 : "memory");
}

// 8-byte asynchronous global -> shared copy (LDGSTS, L1-allocating) and the wait for all of them.
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Order this thread's generic-proxy global writes before later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// generic-proxy shared-memory accesses of this thread ordered before later async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Flags shared by a producer warp and the compute warps, which share no barrier: every access is a
// shared-memory atomic, so it is one coherent operation (and not a data race for compute-sanitizer).
__device__ __forceinline__ int flag_ld(volatile int *p) { return atomicAdd(const_cast<int *>(p), 0); }
__device__ __forceinline__ void flag_st(volatile int *p, int v) { atomicExch(const_cast<int *>(p), v); }
__device__ __forceinline__ long long flag_ld64(volatile long long *p) {
    return (long long)atomicAdd(reinterpret_cast<unsigned long long *>(const_cast<long long *>(p)), 0ull);
}
__device__ __forceinline__ void flag_st64(volatile long long *p, long long v) {
    atomicExch(reinterpret_cast<unsigned long long *>(const_cast<long long *>(p)), (unsigned long long)v);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace wc

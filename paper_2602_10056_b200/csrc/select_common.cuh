// select_common.cuh -- helpers shared by the two selection kernels (select.cu: sequential RPC;
// select_blocked.cu: blocked RPC).  Product path only.
#pragma once

#include "common.cuh"

namespace wc {

constexpr int kST = 256;  // keys per super-tile (8 warp-tiles of 32 keys)
constexpr int kTK = kST / 32;

constexpr int kCW = 8;                // compute warps
constexpr int kCT = kCW * 32;         // compute threads (= kST: one key per thread in phases B/C)
constexpr int kRPS = 8;               // F rows per ring stage (one per compute warp)
constexpr int kTmaThreads = kCT + 32; // + producer warp
static_assert(kCT == kST, "one compute thread per super-tile key");

__device__ __forceinline__ void cw_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCT) : "memory"); }

__device__ __forceinline__ double cw_sum(double v, double *scratch) {
    const int lane = threadIdx.x & 31, w = warp_index();
    v = warp_sum(v);
    cw_sync();
    if (lane == 0) scratch[w] = v;
    cw_sync();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kCW; ++k) t += scratch[k];
    cw_sync();
    return t;
}

__device__ __forceinline__ double cw_exclusive_scan(double v, double *scratch) {
    const int lane = threadIdx.x & 31, w = warp_index();
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const double wtot = __shfl_sync(0xffffffffu, incl, 31);
    cw_sync();
    if (lane == 0) scratch[w] = wtot;
    cw_sync();
    double off = 0.0;
    for (int k = 0; k < w; ++k) off += scratch[k];
    const double excl = off + (incl - v);
    cw_sync();
    return excl;
}

// Grid-group barrier of the compute threads: bar.sync orders the CTA's writes before thread 0's
// release-add (release is cumulative); the acquire-load orders everything after.  Thread 0 then
// publishes `rounds` (this CTA's F rows complete) to the producer warp.
__device__ __forceinline__ void cw_group_barrier(unsigned *ctr, unsigned count, unsigned epoch,
                                                 volatile int *rounds_done, int rounds) {
    cw_sync();
    if (threadIdx.x == 0) {
        if (count > 1) {
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
            const unsigned target = epoch * count;
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                if (v >= target) break;
                __nanosleep(20);
            }
        } else {
            __threadfence();
        }
        flag_st(rounds_done, rounds);
    }
    cw_sync();
}

// Raw K row of one key kept in registers (issued early, consumed after the pivot is known).
template <typename T, int D> struct KRow {
    static constexpr int kVec = D * (int)sizeof(T) / 16;  // 16-byte vectors per row
    static constexpr int kEl = 16 / (int)sizeof(T);        // elements per vector
    uint4 v[kVec];
    __device__ __forceinline__ void load(const T *row) {
        const uint4 *p = reinterpret_cast<const uint4 *>(row);
#pragma unroll
        for (int q = 0; q < kVec; ++q) v[q] = __ldg(p + q);
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int q = 0; q < kVec; ++q) v[q] = make_uint4(0, 0, 0, 0);
    }
    // part[e % 4] += k_j * kc_j over the row (fp64, exact widening of k)
    __device__ __forceinline__ void dot(const double *kc, double part[4]) const { dot_range<0, kVec>(kc, part); }
    // vectors [Q0, Q1) only (compile-time range: the row stays in registers)
    template <int Q0, int Q1> __device__ __forceinline__ void dot_range(const double *kc, double part[4]) const {
#pragma unroll
        for (int q = Q0; q < Q1; ++q) {
            const uint32_t wd[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
            if constexpr (sizeof(T) == 2) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint32_t bits = (e & 1) ? (wd[e >> 1] & 0xffff0000u) : (wd[e >> 1] << 16);
                    part[e & 3] = fma((double)__uint_as_float(bits), kc[q * 8 + e], part[e & 3]);
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) part[e] = fma((double)__uint_as_float(wd[e]), kc[q * 4 + e], part[e]);
            }
        }
    }
};


}  // namespace wc

// axb_iter.cu — the per-iteration kernels of the B200 row-action solver.
//
// One Kaczmarz iteration of the reference (Solver::step, solver.hpp:321-333 →
// select_* :197-258 + update_row :264-318) is three kernels here, captured into
// a CUDA graph by the host:
//
//   K4  k_yg   y = B·R_iᵀ (q row dots, solver.hpp:270) and, when G = A·Aᵀ is not
//              cached, g = A·A_iᵀ (m row dots, the G column of :294).
//   K4b k_zx   z = yᵀ·B (= R_i·BᵀB, :293, as two GEMVs over B — cheaper than the
//              reference's cached n×n BᵀB) fused with K5, the X row update
//              X_t += (coef·A_it)·y (:272-289) and the fresh ‖X−X_ref‖² sum.
//   K2  k_r    the fused residual update: ONE pass over R with 128-bit loads,
//              R_l −= (coef·g_l)·z, ‖R_l‖² emitted in the same pass (:294-305),
//              per-CTA {Σ‖R_l‖², max ratio, argmax} records; the last CTA to
//              finish reduces them, runs the stop/divergence logic (:306-307,
//              :351-358) and — K3 — selects the next row on the device with the
//              reference's xoshiro256** stream (rng.hpp:30-43, 84-99), so no host
//              round trip happens between iterations.
//
// All reductions use fixed shapes and fixed orders: results are deterministic
// run to run.  The R and X updates use separately rounded multiply and subtract
// (__dmul_rn/__dsub_rn), i.e. the reference's arithmetic (no FMA contraction).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>

#include <cooperative_groups.h>

#include "axb_device.cuh"

namespace axb_dev {

#ifdef AXB_CHECKED
__device__ unsigned long long g_axb_violation = 0ull;
unsigned long long checked_violation() {
    unsigned long long v = 0ull, z = 0ull;
    cudaMemcpyFromSymbol(&v, g_axb_violation, sizeof v);
    if (v) cudaMemcpyToSymbol(g_axb_violation, &z, sizeof z);
    return v;
}
#else
unsigned long long checked_violation() { return 0ull; }
#endif

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
static_assert(kWarps == kZxWarps, "k_zx geometry assumes kZxWarps warps per CTA");

// Programmatic dependent launch: the iteration kernels are launched with the
// programmatic-stream-serialization attribute so the next kernel's CTAs are
// scheduled while this one drains; griddepcontrol.wait then blocks until the
// predecessor grid has completed and its writes are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// phase timestamps of the greedy selection into DevState::dbg (build with
// -DAXB_TRACE_SELECT; read with axb_solver_debug_state, tools/sel_timing.py)
#if defined(AXB_TRACE_SELECT) || defined(AXB_TRACE_TIMELINE)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif
#ifdef AXB_TRACE_SELECT
#define AXB_STAMP(slot) (st->dbg[slot] = gtime())
#else
#define AXB_STAMP(slot) ((void)0)
#endif

// In-pipeline timeline of the graph path's iteration kernels (build with
// -DAXB_TRACE_TIMELINE; read with axb_debug_timeline, tools/timeline.py): per
// iteration (ring of 64) the earliest CTA start after its dependency wait and the
// latest CTA end of K4 (0), K4b+K5 (1), K2 (2) and K3 k_sel_greedy (3).  Device
// clock (globaltimer), so it shows what events cannot: the programmatic overlap.
#ifdef AXB_TRACE_TIMELINE
__device__ unsigned long long g_axb_tl[64][8];
#define TL_BEGIN(id, back)                                              \
    const unsigned tl_slot = (unsigned)((P.st->k - (back)) & 63u);       \
    if (threadIdx.x == 0) atomicMin(&g_axb_tl[tl_slot][2 * (id)], gtime())
#define TL_END(id) \
    do { if (threadIdx.x == 0) atomicMax(&g_axb_tl[tl_slot][2 * (id) + 1], gtime()); } while (0)
#else
#define TL_BEGIN(id, back) ((void)0)
#define TL_END(id) ((void)0)
#endif

__device__ __forceinline__ bool halted(const DevState* st) {
    return st->status != ST_RUN || st->k >= st->k_limit;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide sum (deterministic tree); result valid in all threads
__device__ double block_sum(double v, double* red) {  // red: ≥ blockDim.x/32 slots
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
    t = warp_sum(t);
    return t;
}

// (max ratio, smallest index) pair reduction; valid in all threads
__device__ __forceinline__ void maxidx_merge(double& v, long long& i, double ov, long long oi) {
    if (ov > v || (ov == v && oi < i)) {
        v = ov;
        i = oi;
    }
}

__device__ void block_maxidx(double& v, long long& i, double* redv, long long* redi) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        long long oi = __shfl_xor_sync(0xffffffffu, i, o);
        maxidx_merge(v, i, ov, oi);
    }
    __syncthreads();
    if (lane == 0) {
        redv[w] = v;
        redi[w] = i;
    }
    __syncthreads();
    v = -INFINITY;
    i = LLONG_MAX;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) maxidx_merge(v, i, redv[k], redi[k]);
}

// ---- xoshiro256** (rng.hpp:30-43) ----
__device__ __forceinline__ unsigned long long rotl64(unsigned long long x, int k) {
    return (x << k) | (x >> (64 - k));
}
__device__ unsigned long long rng_next(unsigned long long* s) {
    const unsigned long long result = rotl64(s[1] * 5ull, 7) * 9ull;
    const unsigned long long t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}
__device__ double rng_unit(unsigned long long* s) {
    return __dmul_rn((double)(rng_next(s) >> 11), 0x1.0p-53);
}

// dot of a row with a vector by one warp; lane-strided partials then a
// shuffle tree (deterministic).  vec2: both pointers 16-byte aligned, len even.
// coherent_v: v is written inside the running kernel (R_i in the persistent
// kernel), so it is read through L2 (ld.cg) instead of the non-coherent path.
__device__ double warp_dot(const double* __restrict__ row, const double* __restrict__ v,
                           long long len, int lane, bool vec2, bool coherent_v = false) {
    double acc = 0.0;
    if (vec2) {
        const double2* r2 = reinterpret_cast<const double2*>(row);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const long long h = len >> 1;
#pragma unroll 4
        for (long long k = lane; k < h; k += 32) {
            const double2 a = __ldg(r2 + k);
            const double2 b = coherent_v ? __ldcg(v2 + k) : __ldg(v2 + k);
            acc += a.x * b.x;
            acc += a.y * b.y;
        }
    } else {
#pragma unroll 4
        for (long long k = lane; k < len; k += 32)
            acc += __ldg(row + k) * (coherent_v ? __ldcg(v + k) : __ldg(v + k));
    }
    return warp_sum(acc);
}

// two row dots against one vector by one warp (row1 may be null): the vector
// segment is loaded once for both rows; per row the same lane-strided partials
// and shuffle tree as warp_dot.
__device__ void warp_dot_pair(const double* __restrict__ row0, const double* __restrict__ row1,
                              const double* __restrict__ v, long long len, int lane, bool vec2,
                              bool coherent_v, double& out0, double& out1) {
    double acc0 = 0.0, acc1 = 0.0;
    const bool two = row1 != nullptr;
    if (vec2) {
        const double2* r0 = reinterpret_cast<const double2*>(row0);
        const double2* r1 = reinterpret_cast<const double2*>(two ? row1 : row0);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const long long h = len >> 1;
#pragma unroll 4
        for (long long k = lane; k < h; k += 32) {
            const double2 b = coherent_v ? __ldcg(v2 + k) : __ldg(v2 + k);
            const double2 a = __ldg(r0 + k);
            acc0 += a.x * b.x;
            acc0 += a.y * b.y;
            if (two) {
                const double2 c = __ldg(r1 + k);
                acc1 += c.x * b.x;
                acc1 += c.y * b.y;
            }
        }
    } else {
#pragma unroll 4
        for (long long k = lane; k < len; k += 32) {
            const double b = coherent_v ? __ldcg(v + k) : __ldg(v + k);
            acc0 += __ldg(row0 + k) * b;
            if (two) acc1 += __ldg(row1 + k) * b;
        }
    }
    out0 = warp_sum(acc0);
    out1 = two ? warp_sum(acc1) : 0.0;
}

// warp_dot_pair with kU vector loads per lane issued before the FMAs (one L2
// round trip per 32·kU elements instead of per 32·4)
template <int kU>
__device__ void warp_dot_pair_u(const double* __restrict__ row0, const double* __restrict__ row1,
                                const double* __restrict__ v, long long len, int lane, bool vec2,
                                bool coherent_v, double& out0, double& out1) {
    double acc0 = 0.0, acc1 = 0.0;
    const bool two = row1 != nullptr;
    if (vec2) {
        const double2* r0 = reinterpret_cast<const double2*>(row0);
        const double2* r1 = reinterpret_cast<const double2*>(two ? row1 : row0);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const long long h = len >> 1;
        for (long long k0 = lane; k0 < h; k0 += 32 * kU) {
            double2 a[kU], b[kU], c[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const long long k = k0 + 32 * u;
                if (k < h) {
                    b[u] = coherent_v ? __ldcg(v2 + k) : __ldg(v2 + k);
                    a[u] = __ldg(r0 + k);
                    if (two) c[u] = __ldg(r1 + k);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const long long k = k0 + 32 * u;
                if (k < h) {
                    acc0 += a[u].x * b[u].x;
                    acc0 += a[u].y * b[u].y;
                    if (two) {
                        acc1 += c[u].x * b[u].x;
                        acc1 += c[u].y * b[u].y;
                    }
                }
            }
        }
    } else {
        for (long long k0 = lane; k0 < len; k0 += 32 * kU) {
            double a[kU], b[kU], c[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const long long k = k0 + 32 * u;
                if (k < len) {
                    b[u] = coherent_v ? __ldcg(v + k) : __ldg(v + k);
                    a[u] = __ldg(row0 + k);
                    if (two) c[u] = __ldg(row1 + k);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const long long k = k0 + 32 * u;
                if (k < len) {
                    acc0 += a[u] * b[u];
                    if (two) acc1 += c[u] * b[u];
                }
            }
        }
    }
    out0 = warp_sum(acc0);
    out1 = two ? warp_sum(acc1) : 0.0;
}

// CSR A: one 32·kXS-column segment of X_t += f·y with the reference's incremental
// error term Σ_j (d1² − d0²) (solver.hpp:272-289), all loads of the segment issued
// before the arithmetic (one L2 round trip per segment).  Per lane the columns
// ascend, every product and sum is separately rounded.
constexpr int kXS = 8;
__device__ __forceinline__ double x_segment_inc(double* __restrict__ xr, const double* __restrict__ rr,
                                                const double* __restrict__ yb, long long q,
                                                long long seg, double f, int lane) {
    const long long k0 = seg * (32 * kXS) + lane;
    double xv[kXS], yv[kXS], rv[kXS];
#pragma unroll
    for (int u = 0; u < kXS; ++u) {
        const long long k = k0 + 32 * u;
        if (k < q) {
            xv[u] = xr[k];
            yv[u] = __ldcg(yb + k);
            rv[u] = rr ? rr[k] : 0.0;
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < kXS; ++u) {
        const long long k = k0 + 32 * u;
        if (k < q) {
            const double x1 = __dadd_rn(xv[u], __dmul_rn(f, yv[u]));
            xr[k] = x1;
            if (rr) {
                const double d0 = __dsub_rn(xv[u], rv[u]), d1 = __dsub_rn(x1, rv[u]);
                acc += __dsub_rn(__dmul_rn(d1, d1), __dmul_rn(d0, d0));
            }
        }
    }
    return acc;
}

// the same behind a call: the latency body sits at the 255-register cap, and
// inlining the segment's 24 staged loads there spills inside its phases
__device__ __noinline__ double x_segment_inc_call(double* xr, const double* rr, const double* yb,
                                                  long long q, long long seg, double f, int lane) {
    return x_segment_inc(xr, rr, yb, q, seg, f, lane);
}

// one row dot with kU vector loads per lane issued before the FMAs (the single-row
// form of warp_dot_pair_u: same per-lane order, two thirds of its registers)
template <int kU>
__device__ __forceinline__ double warp_dot_u(const double* __restrict__ row, const double* __restrict__ v,
                                             long long len, int lane, bool vec2, bool coherent_v) {
    double acc = 0.0;
    if (vec2) {
        const double2* r0 = reinterpret_cast<const double2*>(row);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const long long h = len >> 1;
        for (long long k0 = lane; k0 < h; k0 += 32 * kU) {
            double2 a[kU], b[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const long long k = k0 + 32 * u;
                if (k < h) {
                    b[u] = coherent_v ? __ldcg(v2 + k) : __ldg(v2 + k);
                    a[u] = __ldg(r0 + k);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const long long k = k0 + 32 * u;
                if (k < h) {
                    acc += a[u].x * b[u].x;
                    acc += a[u].y * b[u].y;
                }
            }
        }
    } else {
        for (long long k = lane; k < len; k += 32)
            acc += __ldg(row + k) * (coherent_v ? __ldcg(v + k) : __ldg(v + k));
    }
    return warp_sum(acc);
}

// ------------------------------------------------------------------------
// K4: y = B·R_iᵀ (solver.hpp:270) [+ g = A·A_iᵀ, the Gram column of :294].
// A CTA computes 8 row dots (one per warp) against the shared vector, which is
// staged through shared memory in kYgSeg-column segments, so R_i (A_i) is read
// from L2 once per 8 rows instead of once per row.  Each lane accumulates its
// columns in order across segments, then a shuffle tree: deterministic, and the
// same order as one pass over the row.
constexpr int kYgThreads = 256;
constexpr int kYgWarps = kYgThreads / 32;
constexpr int kYgSeg = 2048;
// rows per CTA (1, 2, 4 or 8: Params::yg_rbq / yg_rbm) are chosen on the host
// (axb_solver.cu): enough CTAs to cover the chip, as many rows as possible per
// staged segment of the shared vector
__global__ void __launch_bounds__(kYgThreads) k_yg(Params P, int with_g) {
    __shared__ __align__(16) double vs[kYgSeg];
    __shared__ double part[kYgWarps];
    if (P.yg_pf && (long long)blockIdx.x * P.yg_rbq < P.q) {
        // B does not depend on the selected row: while the selection this launch
        // waits on finishes (HBM otherwise idle), pull the head of this CTA's
        // first B rows — the part its first segment reads — into L2
        const int rb = P.yg_rbq;
        const long long len8 = 8 * (P.c1 - P.c0);
        const long long per = min(len8, (long long)(P.yg_pf / rb)) & ~4095LL;
        const int cpr = (int)(per >> 12);  // 4 KB pieces per row
        if (cpr > 0 && ((8 * (P.n | P.c0)) & 15) == 0) {
            for (int t = threadIdx.x; t < rb * cpr; t += kYgThreads) {
                const long long it = (long long)blockIdx.x * rb + t / cpr;
                if (it >= P.q) break;
                const char* src = reinterpret_cast<const char*>(P.B + it * P.n + P.c0) +
                                  (long long)(t % cpr) * 4096;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(src) : "memory");
            }
        }
    }
    pdl_wait();
    pdl_trigger();
    const DevState* st = P.st;
    if (halted(st)) return;
    const double* Ri;
    const double* Ai;
    if (P.pack) {  // sharded: the owner's row arrived through the allreduce
        Ri = P.pack;
        Ai = P.pack + P.n;
    } else {
        const long long il = st->sel - P.row0;
        AXB_CHECK(il >= 0 && il < P.m);
        Ri = P.R + il * P.n;
        Ai = P.A + il * P.p;
    }
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int rbq = P.yg_rbq, rbm = P.yg_rbm;
    const long long nbq = (P.q + rbq - 1) / rbq;
    const long long nb = nbq + (with_g ? (P.m + rbm - 1) / rbm : 0);
    for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
        const bool isB = b < nbq;
        const int rb = isB ? rbq : rbm;
        const int wpr = kYgWarps / rb;  // warps per row
        const int r = w / wpr, pw = w % wpr;
        const long long it = isB ? b * rb + r : (b - nbq) * rb + r;
        const long long rows = isB ? P.q : P.m;
        const double* row = isB ? P.B + it * P.n + P.c0 : P.A + it * P.p;
        const double* v = isB ? Ri + P.c0 : Ai;
        const long long len = isB ? P.c1 - P.c0 : P.p;
        const bool live = it < rows;
        const bool v2 = (len & 1) == 0 && ((reinterpret_cast<uintptr_t>(row) |
                                            reinterpret_cast<uintptr_t>(v)) & 15) == 0;
        if (rb == 1) {
            // one row per CTA: no reuse to stage for; all 256 threads stride the
            // row, the vector comes through L1, fixed-order block reduction
            double a0 = 0.0, a1 = 0.0;
            if (live) {
                if (v2) {
                    const double2* r2 = reinterpret_cast<const double2*>(row);
                    const double2* s2 = reinterpret_cast<const double2*>(v);
#pragma unroll 8
                    for (long long k = tid; k < (len >> 1); k += kYgThreads) {
                        const double2 a = __ldg(r2 + k);
                        const double2 bb = __ldg(s2 + k);
                        a0 += a.x * bb.x;
                        a1 += a.y * bb.y;
                    }
                } else {
#pragma unroll 8
                    for (long long k = tid; k < len; k += kYgThreads) a0 += __ldg(row + k) * __ldg(v + k);
                }
            }
            const double t = block_sum(a0 + a1, part);
            if (live && tid == 0) {
                if (isB) P.y[it] = t;
                else P.g[it] = t;
            }
            __syncthreads();
            continue;
        }
        double acc = 0.0;
        for (long long c0 = 0; c0 < len; c0 += kYgSeg) {
            const int sw = (int)min((long long)kYgSeg, len - c0);
            __syncthreads();
            for (int k = tid; k < sw; k += kYgThreads) vs[k] = __ldg(v + c0 + k);
            __syncthreads();
            if (!live) continue;
            // this warp's contiguous share of the segment (multiples of 64 columns)
            const int chunk = (((sw + wpr - 1) / wpr) + 63) & ~63;
            const int k0 = pw * chunk, k1 = min(sw, k0 + chunk);
            if (v2) {
                const double2* r2 = reinterpret_cast<const double2*>(row + c0);
                const double2* s2 = reinterpret_cast<const double2*>(vs);
#pragma unroll 8
                for (int k = (k0 >> 1) + lane; k < (k1 >> 1); k += 32) {
                    const double2 a = __ldg(r2 + k);  // keep B in L2 for the z pass
                    const double2 bb = s2[k];
                    acc += a.x * bb.x;
                    acc += a.y * bb.y;
                }
            } else {
#pragma unroll 8
                for (int k = k0 + lane; k < k1; k += 32) acc += __ldg(row + c0 + k) * vs[k];
            }
        }
        acc = warp_sum(acc);
        __syncthreads();
        if (lane == 0) part[w] = acc;
        __syncthreads();
        if (live && pw == 0 && lane == 0) {  // fixed-order combine of the row's warps
            double t = 0.0;
            for (int k = 0; k < wpr; ++k) t += part[r * wpr + k];
            if (isB) P.y[it] = t;
            else P.g[it] = t;
        }
    }
}

// ------------------------------------------------------------------------
// K4b + K5: z = yᵀ·B (column slabs × row chunks, deterministic last-block
// combine) and the X row update with the fresh ‖X − X_ref‖² partial sums.
constexpr int kZxYStage = 512;  // y entries of one row chunk staged in shared memory
__global__ void __launch_bounds__(kThreads, 4) k_zx(Params P) {
    __shared__ double red[kWarps];
    __shared__ bool last;
    __shared__ double ys[kZxYStage];
    pdl_wait();
    pdl_trigger();
    DevState* st = P.st;
    if (halted(st)) return;
    TL_BEGIN(1, 0);
    const int tid = threadIdx.x;
    // CTAs [0, x_ctas) update X (the larger units, dispatched first), the rest
    // form z — small slab × row-chunk units that even out the tail
    if ((int)blockIdx.x >= P.x_ctas) {
        const int zb = (int)blockIdx.x - P.x_ctas;
        const int slab = zb % P.z_nslab;
        const int jc = zb / P.z_nslab;
        const long long j0 = (long long)jc * P.z_jrows;
        const long long j1 = min(P.q, j0 + P.z_jrows);
        const long long c = P.c0 + (long long)slab * (2 * kThreads) + 2 * tid;
        const long long cend = P.c1;
        // the chunk's y once into shared memory (broadcast reads below)
        const bool ystage = j1 - j0 <= kZxYStage;
        if (ystage) {
            for (long long j = j0 + tid; j < j1; j += kThreads) ys[j - j0] = __ldg(P.y + j);
            __syncthreads();
        }
        auto yat = [&](long long j) { return ystage ? ys[j - j0] : __ldg(P.y + j); };
        double a0 = 0.0, a1 = 0.0;
        if ((P.n & 1) == 0) {
            if (c < cend) {
                const double2* Bc = reinterpret_cast<const double2*>(P.B + c);
                const long long ld2 = P.n >> 1;
                long long j = j0;
                // 8 rows of B in flight per thread: all loads first, then the
                // FMAs in row order (same sums as the one-row loop)
                for (; j + 8 <= j1; j += 8) {
                    double2 b[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) b[u] = __ldcs(Bc + (j + u) * ld2);  // last use of B
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double yv = yat(j + u);
                        a0 += yv * b[u].x;
                        a1 += yv * b[u].y;
                    }
                }
                for (; j < j1; ++j) {
                    const double yj = yat(j);
                    const double2 b = __ldcs(Bc + j * ld2);
                    a0 += yj * b.x;
                    a1 += yj * b.y;
                }
            }
        } else {
            for (long long j = j0; j < j1; ++j) {
                const double yj = yat(j);
                if (c < cend) a0 += yj * __ldg(P.B + j * P.n + c);
                if (c + 1 < cend) a1 += yj * __ldg(P.B + j * P.n + c + 1);
            }
        }
        if (P.z_nj == 1) {
            if (c < cend) P.z[c] = a0;
            if (c + 1 < cend) P.z[c + 1] = a1;
            TL_END(1);
            return;
        }
        double* zp = P.zpart + (long long)jc * P.n;
        if (c < cend) zp[c] = a0;
        if (c + 1 < cend) zp[c + 1] = a1;
        __threadfence();
        __syncthreads();
        if (tid == 0) last = atomicAdd(P.zcnt + slab, 1u) == (unsigned)(P.z_nj - 1);
        __syncthreads();
        TL_END(1);
        if (!last) return;
        __threadfence();
        for (long long cc = c; cc < c + 2 && cc < cend; ++cc) {
            double s = 0.0;
            for (int k = 0; k < P.z_nj; ++k) s += __ldcg(P.zpart + (long long)k * P.n + cc);
            P.z[cc] = s;
        }
        if (tid == 0) P.zcnt[slab] = 0u;
        TL_END(1);
        return;
    }
    // ---- X update (solver.hpp:272-290): one warp per row t of X ----
    const int xb = blockIdx.x;
    const double* Ai = P.pack ? P.pack + P.n : P.A + (st->sel - P.row0) * P.p;
    const double coef = P.pack ? P.pack[P.n + P.p + 1] : st->coef;
    const bool track = P.Xref != nullptr;
    const int lane = tid & 31, warp = tid >> 5;
    const long long q = P.q;
    double acc = 0.0;
    for (long long t = P.x0r + (long long)xb * kWarps + warp; t < P.x1r;
         t += (long long)P.x_ctas * kWarps) {
        const double f = __dmul_rn(coef, __ldg(Ai + t));
        // A_it = 0 leaves X_t unchanged: the reference's loop over the stored
        // entries of A_i (solver.hpp:272-273); skipped unless ‖X−X_ref‖² needs the row
        if (f == 0.0 && !track) continue;
        double* xr = P.X + t * q;
        const double* rr = track ? P.Xref + t * q : nullptr;
        if ((q & 1) == 0) {
            double2* x2 = reinterpret_cast<double2*>(xr);
            const double2* y2 = reinterpret_cast<const double2*>(P.y);
            const double2* f2 = reinterpret_cast<const double2*>(rr);
            const long long h = q >> 1;
            long long k = lane;
            // 4 segments per lane in flight: loads first, then update + store
            for (; k + 96 < h; k += 128) {
                double2 x[4], yy[4], rf[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    x[u] = x2[k + 32 * u];
                    yy[u] = __ldg(y2 + k + 32 * u);
                    if (track) rf[u] = __ldg(f2 + k + 32 * u);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    x[u].x = __dadd_rn(x[u].x, __dmul_rn(f, yy[u].x));
                    x[u].y = __dadd_rn(x[u].y, __dmul_rn(f, yy[u].y));
                    x2[k + 32 * u] = x[u];
                    if (track) {
                        const double d0 = x[u].x - rf[u].x, d1 = x[u].y - rf[u].y;
                        acc += d0 * d0 + d1 * d1;
                    }
                }
            }
            for (; k < h; k += 32) {
                double2 x = x2[k];
                const double2 yy = __ldg(y2 + k);
                x.x = __dadd_rn(x.x, __dmul_rn(f, yy.x));
                x.y = __dadd_rn(x.y, __dmul_rn(f, yy.y));
                x2[k] = x;
                if (track) {
                    const double2 rf = __ldg(f2 + k);
                    const double d0 = x.x - rf.x, d1 = x.y - rf.y;
                    acc += d0 * d0 + d1 * d1;
                }
            }
        } else {
            for (long long k = lane; k < q; k += 32) {
                const double x1 = __dadd_rn(xr[k], __dmul_rn(f, __ldg(P.y + k)));
                xr[k] = x1;
                if (track) {
                    const double d1 = x1 - __ldg(rr + k);
                    acc += d1 * d1;
                }
            }
        }
    }
    TL_END(1);
    if (!track) return;
    acc = block_sum(acc, red);
    if (tid == 0) {
        P.xpart[xb] = acc;
        __threadfence();
        last = atomicAdd(&st->cnt_x, 1u) == (unsigned)(P.x_ctas - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0.0;
    for (int k = tid; k < P.x_ctas; k += kThreads) s += __ldcg(P.xpart + k);
    s = block_sum(s, red);
    if (tid == 0) {
        st->err_sq = s;
        st->cnt_x = 0u;
    }
    TL_END(1);
}

// ------------------------------------------------------------------------
// K3: row selection for the next iteration, executed by one 256-thread block.
// Writes *out_row; returns an axb_status (0 ok).  All threads must call it.
struct SelShared {
#ifdef AXB_TRACE_PERSIST
    unsigned long long t_groups;  // globaltimer after the greedy group sums
#endif
    double scan[kThreads];
    double redv[32];  // per-warp slots for blocks of up to 1024 threads
    long long redi[32];
    double target;
    double u;
    long long cand;
    int err;
};

// ---- greedy membership and the two-level member-mass scan ----------------
// member mass of local row i (r_sq) when it belongs to the greedy index set
// 𝒥_k (solver.hpp:226-237), else −1.  ζ follows solver.hpp:215 with separately
// rounded operations; the argmax row is a member by construction.
struct Member {
    const double* a_sq;
    const double* r_sq;
    long long row0, argmax;
    double zeta, r_fro;
    int smem;  // a_sq / r_sq point at shared-memory copies (persistent kernel)
    __device__ double rs_at(long long i) const { return smem ? r_sq[i] : __ldcg(r_sq + i); }
    __device__ double operator()(long long i) const {
        const double as = a_sq[i];
        if (as <= 0.0) return -1.0;
        const double rs = rs_at(i);
        return (row0 + i == argmax || rs >= __dmul_rn(__dmul_rn(zeta, as), r_fro)) ? rs : -1.0;
    }
};

__device__ Member make_member(const Params& P, const DevState* st, double theta) {
    Member mm;
    mm.a_sq = P.a_sq;
    mm.r_sq = P.r_sq;
    mm.smem = 0;
    mm.row0 = P.row0;
    mm.argmax = st->argmax;
    mm.r_fro = st->r_fro_sq;
    mm.zeta = __dadd_rn(__dmul_rn(theta, __ddiv_rn(st->max_ratio, mm.r_fro)),
                        __ddiv_rn(__dsub_rn(1.0, theta), P.a_fro_sq));
    return mm;
}

// gs[g] = Σ member masses of rows [32g, 32g+32) for g in [g_begin, g_end):
// coalesced, branch-free loads (8 groups × 2 arrays in flight per warp, every
// warp of the block), warp trees.  A group's sum does not depend on which CTA
// forms it, so one CTA (K2's last) or many (k_sel_greedy) give identical gs.
__device__ void grbk_group_sums(const Member& mem, long long m, double* gs,
                                long long g_begin = 0, long long g_end = -1) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (int)(blockDim.x >> 5);
    const long long ng = g_end < 0 ? (m + 31) / 32 : g_end;
    constexpr int kG = 8;
    for (long long gb = g_begin + warp; gb < ng; gb += (long long)nw * kG) {
        double as[kG], rs[kG];
#pragma unroll
        for (int u = 0; u < kG; ++u) {
            const long long g = gb + (long long)u * nw;
            const long long i = g * 32 + lane;
            const bool ok = g < ng && i < m;
            as[u] = ok ? mem.a_sq[i] : 0.0;
            rs[u] = ok ? mem.rs_at(i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kG; ++u) {
            const long long g = gb + (long long)u * nw;
            if (g >= ng) break;  // warp-uniform
            const long long i = g * 32 + lane;
            const bool member =
                as[u] > 0.0 && (mem.row0 + i == mem.argmax ||
                                rs[u] >= __dmul_rn(__dmul_rn(mem.zeta, as[u]), mem.r_fro));
            const double v = warp_sum(member ? rs[u] : 0.0);
            AXB_CHECK(g >= 0 && g < (m + 31) / 32);
            if (lane == 0) gs[g] = v;
        }
    }
    __syncthreads();
}

// ordered inclusive prefix over gs: contiguous runs per thread, Hillis–Steele
// across the runs (fixed order → deterministic).  Returns the total; [g0, g1)
// and excl describe the calling thread's run.
__device__ double grbk_prefix(const double* gs, long long ng, SelShared& sh, long long& g0,
                              long long& g1, double& excl) {
    const int tid = threadIdx.x;
    const bool scan_lane = tid < kThreads;  // blocks may carry an extra producer warp
    const long long gseg = (ng + kThreads - 1) / kThreads;
    g0 = scan_lane ? min(ng, (long long)tid * gseg) : ng;
    g1 = min(ng, g0 + gseg);
    double local = 0.0;
    for (long long g = g0; g < g1; ++g) local = __dadd_rn(local, gs[g]);
    if (scan_lane) sh.scan[tid] = local;
    __syncthreads();
    for (int off = 1; off < kThreads; off <<= 1) {
        const double v = (scan_lane && tid >= off) ? sh.scan[tid - off] : 0.0;
        __syncthreads();
        if (scan_lane) sh.scan[tid] = __dadd_rn(sh.scan[tid], v);
        __syncthreads();
    }
    excl = (scan_lane && tid) ? sh.scan[tid - 1] : 0.0;
    const double total = sh.scan[kThreads - 1];
    __syncthreads();
    return total;
}

// First local row whose cumulative member mass (thread prefixes `excl`, which
// may include a cross-shard base) exceeds target.  Returns −1 when the draw
// lands within `slack` of a boundary (slack ≥ 0) or the two rounding paths
// disagree — the caller then falls back to an exact sequential walk.
__device__ long long grbk_search(const Member& mem, long long m, const double* gs, long long g0,
                                 long long g1, double excl, double target, double slack,
                                 SelShared& sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        sh.cand = LLONG_MAX;
        sh.err = 0;
    }
    __syncthreads();
    long long my_g = LLONG_MAX;
    double my_before = 0.0;
    {
        double cum = excl;
        for (long long g = g0; g < g1; ++g) {
            const double nc = __dadd_rn(cum, gs[g]);
            if (nc > target) {
                my_g = g;
                my_before = cum;
                break;
            }
            cum = nc;
        }
        if (my_g != LLONG_MAX)
            atomicMin(reinterpret_cast<unsigned long long*>(&sh.cand), (unsigned long long)my_g);
    }
    __syncthreads();
    const long long G = sh.cand;
    if (my_g == G && G != LLONG_MAX) sh.redv[0] = my_before;  // unique owner of G
    __syncthreads();
    if (G != LLONG_MAX && warp == 0) {
        // within group G: lane-inclusive scan of the member masses
        const long long i = G * 32 + lane;
        const double w = (i < m) ? mem(i) : -1.0;
        double v = w > 0.0 ? w : 0.0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off) v = __dadd_rn(v, t);
        }
        const double before = sh.redv[0];  // cumulative mass before group G
        const double cum = __dadd_rn(before, v);
        double prev = __shfl_up_sync(0xffffffffu, cum, 1);
        if (lane == 0) prev = before;
        const unsigned hit = __ballot_sync(0xffffffffu, w >= 0.0 && cum > target);
        if (hit == 0u) {
            if (lane == 0) sh.err = -1;  // the two rounding paths disagree
        } else {
            const int first = __ffs(hit) - 1;
            const double hi = __shfl_sync(0xffffffffu, cum, first);
            const double lo = __shfl_sync(0xffffffffu, prev, first);
            if (lane == 0) {
                sh.cand = G * 32 + first;
                if (slack >= 0.0 && (hi - target <= slack || target - lo <= slack)) sh.err = -1;
            }
        }
    }
    __syncthreads();
    const long long pick = (G == LLONG_MAX || sh.err == -1) ? -1 : sh.cand;
    __syncthreads();
    return pick;
}

__device__ int grbk_pick(const Params& P, DevState* st, const Member& mem, const double* gs,
                         long long m, long long row0, long long* out_row, SelShared& sh);

// Distance from a member-mass boundary inside which the tree-ordered search may
// round differently from the reference's sequential prefix: the draw then takes
// the exact sequential walk.  tie_guard 0 = off, 1 = on (default), 2 = every
// draw takes the walk (a test hook that exercises the near-tie path on every step).
__device__ __forceinline__ double tie_slack(const Params& P, long long m, double total) {
    if (P.tie_guard == 2) return INFINITY;
    return P.tie_guard ? 8.0 * (double)m * DBL_EPSILON * total : -1.0;
}

__device__ int select_rows(const Params& P, DevState* st, int method, double theta,
                           long long* out_row, SelShared& sh, double* scratch,
                           long long scratch_cap, const double* as_sm = nullptr,
                           const double* rs_sm = nullptr, const double* cum_sm = nullptr) {
    const int tid = threadIdx.x;
    const long long m = P.m;
    if (st->replay) {
        // replay of a given index stream (the reference's): consume the same
        // RNG draw / cyclic advance the reference's select_* would, take the row
        if (tid == 0) {
            AXB_CHECK(st->k - st->k0 < P.trace_cap);
            const long long row = P.forced_rows[st->k - st->k0];
            sh.err = (row < 0 || row >= m || !(P.a_sq[row] > 0.0)) ? 2 : 0;
            sh.cand = row;
            if (method == 1 || method == 2 || method == 3) (void)rng_next(st->rng);
            if (method == 0 && !sh.err) st->cyclic_pos = (unsigned long long)((row + 1) % m);
        }
        __syncthreads();
        *out_row = sh.cand;
        return sh.err;
    }
    if (method == 4) {  // MWRBK: smallest argmax (solver.hpp:258, 387-400)
        if (st->argmax == LLONG_MAX) return 2;
        *out_row = st->argmax;
        return 0;
    }
    if (method == 0) {  // BK: cyclic, zero rows skipped (solver.hpp:197-206)
        if (tid == 0) {
            sh.err = 2;
            for (long long tries = 0; tries < m; ++tries) {
                const long long i = (long long)st->cyclic_pos;
                st->cyclic_pos = (st->cyclic_pos + 1) % (unsigned long long)m;
                if (P.a_sq[i] > 0.0) {
                    sh.cand = i;
                    sh.err = 0;
                    break;
                }
                ++st->skipped_zero_rows;
            }
        }
        __syncthreads();
        *out_row = sh.cand;
        return sh.err;
    }
    if (method == 1) {  // RBK: categorical_cdf on the static ‖A_i‖² CDF (solver.hpp:209)
        if (tid == 0) {
            const double* cum = cum_sm ? cum_sm : P.rbk_cum;
            const double total = cum[m - 1];
            sh.err = 0;
            if (!(total > 0.0)) {
                sh.err = 2;
            } else {
                const double target = __dmul_rn(rng_unit(st->rng), total);
                long long lo = 0, hi = m - 1;
                while (lo < hi) {  // rng.hpp:88-95
                    const long long mid = (lo + hi) / 2;
                    if (cum[mid] <= target) lo = mid + 1;
                    else hi = mid;
                }
                while (lo > 0 && cum[lo] == cum[lo - 1]) --lo;  // rng.hpp:97
                sh.cand = lo;
            }
        }
        __syncthreads();
        *out_row = sh.cand;
        return sh.err;
    }
    // GRBK / RGRBK (solver.hpp:212-254): ζ, membership, member-mass draw.
    if (!(st->r_fro_sq > 0.0)) return 2;  // "greedy threshold: zero residual"
    if (tid == 0) AXB_STAMP(0);
    Member mem = make_member(P, st, theta);
    if (as_sm) {
        mem.a_sq = as_sm;
        mem.r_sq = rs_sm;
        mem.smem = 1;
    }
    double* gs = (scratch != nullptr && (m + 31) / 32 <= scratch_cap) ? scratch : P.gsum;
    grbk_group_sums(mem, m, gs);
#ifdef AXB_TRACE_PERSIST
    if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(sh.t_groups));
#endif
    return grbk_pick(P, st, mem, gs, P.m, P.row0, out_row, sh);
}

// The greedy draw once the group sums gs are in place: ordered prefix, one
// uniform, two-level search with the tie guard, exact sequential fallback.
// Up to 1024 groups (m ≤ 32768) the whole draw runs in warp 0 with shuffles —
// contiguous runs of groups per lane, a shuffle scan across the runs, the run
// search, then the in-group rescan — and the block meets at one barrier.  The
// arithmetic is grbk_prefix/grbk_search's with a different (fixed) association
// of the group sums; the tie guard covers the rounding difference exactly as
// it does between those and the reference's sequential walk.
__device__ long long grbk_pick_warp(const Params& P, DevState* st, const Member& mem,
                                    const double* gs, long long m, long long ng, SelShared& sh) {
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) {
        const long long gseg = (ng + 31) / 32;
        const long long g0 = min(ng, (long long)lane * gseg), g1 = min(ng, g0 + gseg);
        double local = 0.0;
        for (long long g = g0; g < g1; ++g) local = __dadd_rn(local, gs[g]);
        double incl = local;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl = __dadd_rn(t, incl);
        }
        const double total = __shfl_sync(0xffffffffu, incl, 31);
        double excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0.0;
        int err = 0;
        long long cand = -1;
        if (!(total > 0.0)) {
            err = 2;  // mass on zero rows only (solver.hpp:249-252)
        } else {
            double u = 0.0;
            if (lane == 0) u = rng_unit(st->rng);
            u = __shfl_sync(0xffffffffu, u, 0);
            const double target = __dmul_rn(u, total);
            const double slack = tie_slack(P, m, total);
            long long my_g = -1;
            double my_before = 0.0, cum = excl;
            for (long long g = g0; g < g1; ++g) {
                const double nc = __dadd_rn(cum, gs[g]);
                if (nc > target) {
                    my_g = g;
                    my_before = cum;
                    break;
                }
                cum = nc;
            }
            const unsigned hitl = __ballot_sync(0xffffffffu, my_g >= 0);
            if (hitl == 0u) {
                err = -1;
            } else {
                const int fl = __ffs(hitl) - 1;
                const long long G = __shfl_sync(0xffffffffu, my_g, fl);
                const double before = __shfl_sync(0xffffffffu, my_before, fl);
                const long long i = G * 32 + lane;
                const double w = (i < m) ? mem(i) : -1.0;
                double v = w > 0.0 ? w : 0.0;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const double t = __shfl_up_sync(0xffffffffu, v, off);
                    if (lane >= off) v = __dadd_rn(v, t);
                }
                const double c = __dadd_rn(before, v);
                double prev = __shfl_up_sync(0xffffffffu, c, 1);
                if (lane == 0) prev = before;
                const unsigned hit = __ballot_sync(0xffffffffu, w >= 0.0 && c > target);
                if (hit == 0u) {
                    err = -1;  // the two rounding paths disagree
                } else {
                    const int first = __ffs(hit) - 1;
                    const double hi = __shfl_sync(0xffffffffu, c, first);
                    const double lo = __shfl_sync(0xffffffffu, prev, first);
                    cand = G * 32 + first;
                    if (slack >= 0.0 && (hi - target <= slack || target - lo <= slack)) err = -1;
                }
            }
            if (lane == 0) sh.u = u;
        }
        if (lane == 0) {
            sh.err = err;
            sh.cand = cand;
        }
    }
    __syncthreads();
    const long long r = sh.err == 2 ? -2 : (sh.err == -1 ? -1 : sh.cand);
    __syncthreads();
    return r;
}

// m rows of mem / gs; the picked row is row0 + its index (K2's shard offset on
// one GPU, 0 for the sharded path's global arrays)
__device__ int grbk_pick(const Params& P, DevState* st, const Member& mem, const double* gs,
                         long long m, long long row0, long long* out_row, SelShared& sh) {
    const int tid = threadIdx.x;
    const long long ng = (m + 31) / 32;
    if (tid == 0) AXB_STAMP(1);
    long long pick;
    if (ng <= 1024) {
        pick = grbk_pick_warp(P, st, mem, gs, m, ng, sh);
        if (tid == 0) AXB_STAMP(2);
        if (pick == -2) return 2;
    } else {
        long long g0, g1;
        double excl;
        const double total = grbk_prefix(gs, ng, sh, g0, g1, excl);
        if (tid == 0) AXB_STAMP(2);
        if (!(total > 0.0)) return 2;  // mass on zero rows only (solver.hpp:249-252)
        if (tid == 0) {
            sh.u = rng_unit(st->rng);
            sh.target = __dmul_rn(sh.u, total);
        }
        __syncthreads();
        const double slack = tie_slack(P, m, total);
        pick = grbk_search(mem, m, gs, g0, g1, excl, sh.target, slack, sh);
    }
    if (tid == 0) {
        AXB_STAMP(3);
        st->dbg[5] += 1;  // selections
        if (pick < 0) st->dbg[6] += 1;  // exact sequential fallbacks
    }
    if (pick < 0) {
        __syncthreads();
        if (tid == 0) {
            // Sequential replay of solver.hpp:243-253 + rng.hpp:84-99 with the same
            // uniform u: cumulative mass in ascending member order, target = u·total,
            // upper_bound, then walk back over a trailing zero-weight plateau.
            const double u = sh.u;
            double total_seq = 0.0;
            for (long long r = 0; r < m; ++r) {
                const double w = mem(r);
                if (w >= 0.0) total_seq = __dadd_rn(total_seq, w);
            }
            const double tseq = __dmul_rn(u, total_seq);
            double cum = 0.0;
            long long found = -1, first_member = -1, last_change = -1;
            for (long long r = 0; r < m && found < 0; ++r) {
                const double w = mem(r);
                if (w < 0.0) continue;
                if (first_member < 0) first_member = r;
                const double nc = __dadd_rn(cum, w);
                if (nc > tseq) found = r;
                if (nc != cum) last_change = r;
                cum = nc;
            }
            if (found < 0) found = last_change >= 0 ? last_change : first_member;
            sh.cand = found;
            atomicAdd(&st->tie_guard_hits, 1);
        }
        __syncthreads();
        pick = sh.cand;
    }
    if (tid == 0) AXB_STAMP(4);
    AXB_CHECK(pick >= 0 && pick < m);
    *out_row = row0 + pick;
    return 0;
}

// snapshot before a speculative pre-selection (rolled back by k_rollback)
__device__ void sel_snapshot(DevState* st, SelShared& sh) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) st->rng_snap[k] = st->rng[k];
        st->cyclic_snap = st->cyclic_pos;
        st->skipped_snap = st->skipped_zero_rows;
        sh.err = 0;
    }
    __syncthreads();
}

__device__ void sel_commit(const Params& P, DevState* st, int err, long long row) {
    if (threadIdx.x == 0) {
        if (err) {
            st->status = ST_ERROR;
            st->err_code = err;
            st->err_k = st->k;
            st->sel_valid = 0;
        } else {
            AXB_CHECK(row - P.row0 >= 0 && row - P.row0 < P.m);
            st->sel = row;
            st->coef = __ddiv_rn(P.alpha, P.a_sq[row - P.row0]);
            st->sel_valid = 1;
        }
    }
}

// block-level finalize + selection shared by k_r's last block and k_select
__device__ void finish_select(const Params& P, DevState* st, SelShared& sh, double* scratch,
                              long long scratch_cap) {
    long long row = 0;
    sel_snapshot(st, sh);
    const int err = select_rows(P, st, P.method, P.theta, &row, sh, scratch, scratch_cap);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (err) {
            st->status = ST_ERROR;
            st->err_code = err;
            st->err_k = st->k;
            st->sel_valid = 0;
        } else {
            st->sel = row;
            st->coef = __ddiv_rn(P.alpha, P.a_sq[row - P.row0]);
            st->sel_valid = 1;
        }
    }
}

// Everything after the streaming pass of K2: write ‖R_l‖², per-CTA records, and
// in the last CTA to finish the fixed-order reduction, the stop / divergence
// logic (solver.hpp:306-307, :347, :351) and K3 for the next iteration.
// rowacc[t] holds ‖R_{r0+t}‖²; all threads of the block must call it.
// Last-CTA finalize of an iteration (or of a norms pass): publish ‖R‖², max ratio
// and argmax, run the divergence / stop logic and pre-select the next row.
template <bool UPDATE>
__device__ void finalize(const Params& P, DevState* st, double s, double mx, long long ax,
                         double* scratch, long long scratch_cap) {
    __shared__ SelShared sh;
    const int tid = threadIdx.x;
    const int mode = UPDATE ? st->fin_mode : FIN_NORMS;
    __syncthreads();
    if (P.pack) {
        // sharded: publish this shard's record; the global reduction, the stop
        // logic and the selection run in k_sel1 after the grouped allgather
        if (tid == 0) {
            st->cnt_r = 0u;
            double* rec = P.recs + 4 * P.rank;
            rec[0] = s;
            rec[1] = mx;
            rec[2] = (double)ax;
            rec[3] = P.Xref ? st->err_sq : 0.0;
        }
        return;
    }
    if (tid == 0) {
        st->cnt_r = 0u;
        st->r_fro_sq = s;
        st->max_ratio = mx;
        st->argmax = ax;
        st->sel_valid = 0;
        const double cf = P.c_fro > 0.0 ? P.c_fro : 1.0;
        const double rel = sqrt(s > 0.0 ? s : 0.0) / cf;
        if (mode != FIN_NORMS && !isfinite(s)) {  // solver.hpp:306-307
            st->status = ST_ERROR;
            st->err_code = 4;
            st->err_k = st->k;
            st->err_val = sqrt(fabs(s));
        } else if (mode == FIN_ITERATION) {
            const unsigned long long k = st->k;
            const double metric = P.stop_kind == 0 ? st->err_sq / P.ref_sq : rel;
            const unsigned long long slot = k - st->k0;
            if (slot < P.trace_cap) {
                P.trace_row[slot] = st->sel;
                P.trace_metric[slot] = metric;
                P.trace_rel[slot] = rel;
            }
            st->k = k + 1;
            st->metric = metric;
            if (st->run_mode && metric <= P.tol) st->status = ST_PAUSE;        // :351
            else if (st->run_mode && !(s > 0.0)) st->status = ST_ZERO;         // :347
        } else {
            st->metric = P.stop_kind == 0 ? st->err_sq / P.ref_sq : rel;
        }
    }
    __syncthreads();
    if (mode == FIN_ITERATION && st->status == ST_RUN && st->k < st->k_limit) {
        if (P.sel_split && (P.method == 2 || P.method == 3) && !st->replay) {
            if (tid == 0) st->sel_pending = 1;  // k_sel_greedy (next launch) selects
        } else {
            finish_select(P, st, sh, scratch, scratch_cap);
        }
    }
}

template <bool UPDATE>
__device__ void r_tail(const Params& P, DevState* st, long long r0, long long r1,
                       const double* rowacc, double* scratch, long long scratch_cap) {
    __shared__ double redv[32];
    __shared__ long long redi[32];
    __shared__ bool last;
    const int tid = threadIdx.x;
    double bsum = 0.0, bmax = -INFINITY;
    long long barg = LLONG_MAX;
    for (long long t = tid; t < r1 - r0; t += blockDim.x) {
        const long long l = r0 + t;
        const double rs = rowacc[t];
        P.r_sq[l] = rs;
        bsum += rs;
        const double as = P.a_sq[l];
        if (as > 0.0) maxidx_merge(bmax, barg, __ddiv_rn(rs, as), P.row0 + l);
    }
    bsum = block_sum(bsum, redv);
    block_maxidx(bmax, barg, redv, redi);
    if (tid == 0) {
        P.rrec[blockIdx.x] = RowRecord{bsum, bmax, barg, 0.0};
        __threadfence();
        last = atomicAdd(&st->cnt_r, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    // ---- last CTA: reduce the records (fixed order), finalize the iteration ----
    __threadfence();
    double s = 0.0, mx = -INFINITY;
    long long ax = LLONG_MAX;
    for (int k = tid; k < (int)gridDim.x; k += blockDim.x) {
        const double* rp = reinterpret_cast<const double*>(P.rrec + k);
        const RowRecord rc{__ldcg(rp), __ldcg(rp + 1), __ldcg(reinterpret_cast<const long long*>(rp + 2)), 0.0};
        s += rc.sum;
        maxidx_merge(mx, ax, rc.max_ratio, rc.argmax);
    }
    s = block_sum(s, redv);
    block_maxidx(mx, ax, redv, redi);
    finalize<UPDATE>(P, st, s, mx, ax, scratch, scratch_cap);
}

// ------------------------------------------------------------------------
// K2: fused residual update + row norms + reductions (+ finalize / K3 select)
template <bool UPDATE, bool VEC2>
__global__ void __launch_bounds__(kThreads) k_r(Params P) {
    extern __shared__ double smem[];
    pdl_wait();
    pdl_trigger();
    DevState* st = P.st;
    if (UPDATE && halted(st)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = P.m, n = P.n;
    const long long r0 = (long long)blockIdx.x * P.r_rows_per_cta;
    const long long r1 = min(m, r0 + P.r_rows_per_cta);
    double* zs = smem;
    double* rowacc = smem + P.r_chunk;
    double coef = 0.0;
    long long sel = 0;
    if (UPDATE) {
        coef = P.pack ? P.pack[P.n + P.p + 1] : st->coef;
        sel = P.pack ? (long long)P.pack[P.n + P.p] : st->sel;
    }
    for (long long t = tid; t < r1 - r0; t += kThreads) rowacc[t] = 0.0;
    for (long long c0 = 0; c0 < n; c0 += P.r_chunk) {
        const long long cw = min((long long)P.r_chunk, n - c0);
        __syncthreads();
        if (UPDATE)
            for (long long t = tid; t < cw; t += kThreads) zs[t] = __ldg(P.z + c0 + t);
        __syncthreads();
        for (long long l = r0 + warp; l < r1; l += kWarps) {
            double f = 0.0;
            if (UPDATE) {
                const double gl = P.G ? __ldg(P.G + sel * m + l) : __ldg(P.g + l);
                f = __dmul_rn(coef, gl);  // solver.hpp:296
            }
            double* row = P.R + l * n + c0;
            double acc = 0.0;
            // explicit batches of kU independent 128-bit loads per lane before any
            // store, so each warp keeps kU×512 B of R in flight (the compiler will
            // not hoist loads across the streaming stores on its own)
            constexpr int kU = 8;
            if (VEC2) {
                double2* r2 = reinterpret_cast<double2*>(row);
                const double2* z2 = reinterpret_cast<const double2*>(zs);
                const long long h = cw >> 1;
                for (long long kb = lane; kb < h; kb += 32 * kU) {
                    double2 rv[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u)
                        if (kb + 32 * u < h) rv[u] = __ldcs(r2 + kb + 32 * u);
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const long long k = kb + 32 * u;
                        if (k < h) {
                            double2 r = rv[u];
                            if (UPDATE) {
                                const double2 zz = z2[k];
                                r.x = __dsub_rn(r.x, __dmul_rn(f, zz.x));  // solver.hpp:300
                                r.y = __dsub_rn(r.y, __dmul_rn(f, zz.y));
                                __stcs(r2 + k, r);
                            }
                            acc += r.x * r.x;  // solver.hpp:301 (tree order here)
                            acc += r.y * r.y;
                        }
                    }
                }
            } else {
                for (long long kb = lane; kb < cw; kb += 32 * kU) {
                    double rv[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u)
                        if (kb + 32 * u < cw) rv[u] = row[kb + 32 * u];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const long long k = kb + 32 * u;
                        if (k < cw) {
                            double r = rv[u];
                            if (UPDATE) {
                                r = __dsub_rn(r, __dmul_rn(f, zs[k]));
                                row[k] = r;
                            }
                            acc += r * r;
                        }
                    }
                }
            }
            acc = warp_sum(acc);
            if (lane == 0) rowacc[l - r0] += acc;
        }
    }
    __syncthreads();
    r_tail<UPDATE>(P, st, r0, r1, rowacc, smem, P.r_chunk);
}

// ------------------------------------------------------------------------
// K2 (even n, the production path): the same fused update, with R streamed
// through shared memory by 1-D bulk TMA copies (cp.async.bulk, SASS UBLKCP) in a
// kTmaStages-deep mbarrier ring.  One producer warp issues the copies; eight
// consumer warps apply R_l −= (coef·g_l)·z from shared memory, write the result
// straight back with streaming stores and accumulate ‖R_l‖².  Each CTA owns a
// contiguous block of rows and walks it in row-major tiles of r_chunk columns,
// so DRAM sees one sequential read stream and one write stream per CTA, and the
// bytes in flight per SM (stages × tile × CTAs) do not depend on registers.
constexpr int kTmaConsumerWarps = 8;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;

__device__ __forceinline__ unsigned smem_u32(const void* ptr) {
    return (unsigned)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    while (!mbar_try(b, parity)) {
    }
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// rows whose warp partials a CTA keeps before a combine flush
constexpr int kRowsKept = 128;

// Fixed-order combine of the kept rows' 8 warp partials (consumer threads only,
// after a consumer barrier): ‖R_l‖² → r_sq, running max / argmax of the ratio.
__device__ void combine_rows(const Params& P, const double* rpart, const long long* rowid, int nkeep,
                             double& cmax, long long& carg) {
    for (int t = threadIdx.x; t < nkeep; t += kTmaConsumerWarps * 32) {
        double a = 0.0;
        for (int w = 0; w < kTmaConsumerWarps; ++w) a += rpart[t * kTmaConsumerWarps + w];
        const long long row = rowid[t];
        AXB_CHECK(row >= 0 && row < P.m);
        P.r_sq[row] = a;
        const double as = P.a_sq[row];
        if (as > 0.0) maxidx_merge(cmax, carg, __ddiv_rn(a, as), P.row0 + row);
    }
}

template <bool UPDATE>
__global__ void __launch_bounds__(kTmaThreads, 2) k_r_tma(Params P) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ long long stage_row[32];
    __shared__ __align__(16) double stage_g[32][2];
    __shared__ double rpart[kRowsKept * kTmaConsumerWarps];
    __shared__ long long rowid[kRowsKept];
    __shared__ double redv[32];
    __shared__ long long redi[32];
    __shared__ bool last;
    pdl_wait();
    pdl_trigger();
    DevState* st = P.st;
    if (UPDATE && halted(st)) return;
    TL_BEGIN(2, 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = P.m, n = P.n;
    const int TW = P.r_chunk;
    const int tpr = (int)((n + TW - 1) / TW);
    const int S = P.r_stages;
    const bool zst = UPDATE && P.r_zstage;  // z segment staged with each tile
    double* stage = reinterpret_cast<double*>(dsm);
    double* zstage = stage + (size_t)S * TW;
    unsigned long long* full =
        reinterpret_cast<unsigned long long*>(dsm + (size_t)S * TW * 8 * (zst ? 2 : 1));
    unsigned long long* empty = full + S;
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kTmaConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double cmax = -INFINITY;
    long long carg = LLONG_MAX;
    long long sel = 0;
    double coef = 0.0;
    if (UPDATE) {
        coef = P.pack ? P.pack[P.n + P.p + 1] : st->coef;
        sel = P.pack ? (long long)P.pack[P.n + P.p] : st->sel;
    }
    if (warp == kTmaConsumerWarps) {
        // ---- producer warp: grab r_grab (≤ 32) rows at a time, read their Gram coefficients
        // coalesced, stream only rows with g ≠ 0 (an exactly-zero coefficient
        // leaves R_l and ‖R_l‖² unchanged — the reference's sparse G iterates
        // stored entries only, solver.hpp:294-295); unchanged rows still enter
        // the max/argmax with their standing ratio ----
        int s = 0;
        unsigned round = 0;
        for (;;) {
            long long base = 0;
            if (lane == 0) base = (long long)atomicAdd(&st->r_next, (unsigned long long)P.r_grab);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base >= m) break;
            const long long row = base + lane;
            const bool valid = lane < P.r_grab && row < m;
            AXB_CHECK(!UPDATE || (sel >= 0 && sel < P.m_global));
            double gl = 0.0;
            bool work = valid;
            if (UPDATE && valid) {
                gl = P.G ? __ldg(P.G + sel * m + row) : __ldg(P.g + row);
                work = gl != 0.0;
                if (!work) {
                    const double as = P.a_sq[row];
                    if (as > 0.0)
                        maxidx_merge(cmax, carg, __ddiv_rn(__ldcg(P.r_sq + row), as), P.row0 + row);
                }
            }
            unsigned mask = __ballot_sync(0xffffffffu, work);
            while (mask) {
                const int l = __ffs(mask) - 1;
                mask &= mask - 1;
                const double g_l = __shfl_sync(0xffffffffu, gl, l);
                if (lane == 0) {
                    const double* src = P.R + (base + l) * n;
                    AXB_CHECK(base + l >= 0 && base + l < m);
                    for (int seg = 0; seg < tpr; ++seg, src += TW) {
                        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
                        stage_row[s] = base + l;
                        stage_g[s][0] = g_l;
                        const unsigned bytes = (unsigned)(min((long long)TW, n - (long long)seg * TW) * 8);
                        mbar_expect_tx(&full[s], bytes * (zst ? 2u : 1u));
                        tma_load_1d(stage + (size_t)s * TW, src, bytes, &full[s]);
                        if (zst)
                            tma_load_1d(zstage + (size_t)s * TW, P.z + (long long)seg * TW, bytes,
                                        &full[s]);
                        if (++s == S) {
                            s = 0;
                            ++round;
                        }
                    }
                }
            }
        }
        if (lane == 0) {  // sentinel: no bytes
            if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
            stage_row[s] = -1;
            mbar_arrive(&full[s]);
        }
    } else {
        // ---- 8 consumer warps ----
        int s = 0, nkeep = 0;
        unsigned round = 0;
        for (;;) {
            mbar_wait(&full[s], round & 1);
            const long long row = stage_row[s];
            if (row < 0) break;
            AXB_CHECK(row < m);
            double f = 0.0;
            if (UPDATE) f = __dmul_rn(coef, stage_g[s][0]);  // solver.hpp:296
            double acc = 0.0;
            long long c0 = 0;
            for (int seg = 0; seg < tpr; ++seg, c0 += TW) {
                if (seg > 0) mbar_wait(&full[s], round & 1);
                const int h = (int)(min((long long)TW, n - c0) >> 1);
                const double2* src = reinterpret_cast<const double2*>(stage + (size_t)s * TW);
                double2* dst = reinterpret_cast<double2*>(P.R + row * n + c0);
                const double2* z2 = zst ? reinterpret_cast<const double2*>(zstage + (size_t)s * TW)
                                        : reinterpret_cast<const double2*>(P.z + c0);
#pragma unroll 4
                for (int k = tid; k < h; k += kTmaConsumerWarps * 32) {
                    double2 r = src[k];
                    if (UPDATE) {
                        const double2 zz = zst ? z2[k] : __ldg(z2 + k);
                        r.x = __dsub_rn(r.x, __dmul_rn(f, zz.x));  // solver.hpp:300
                        r.y = __dsub_rn(r.y, __dmul_rn(f, zz.y));
                        __stcs(dst + k, r);
                    }
                    acc += r.x * r.x;  // solver.hpp:301 (tree order here)
                    acc += r.y * r.y;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (++s == S) {
                    s = 0;
                    ++round;
                }
            }
            // keep this warp's partial of ‖R_row‖²; combined in fixed order later
            acc = warp_sum(acc);
            if (lane == 0) rpart[nkeep * kTmaConsumerWarps + warp] = acc;
            if (tid == 0) rowid[nkeep] = row;
            if (++nkeep == kRowsKept) {  // rare flush (long runs of rows per CTA)
                asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumerWarps * 32) : "memory");
                combine_rows(P, rpart, rowid, nkeep, cmax, carg);
                asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumerWarps * 32) : "memory");
                nkeep = 0;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumerWarps * 32) : "memory");
        combine_rows(P, rpart, rowid, nkeep, cmax, carg);
    }
    // records: max/argmax only (order-independent); ‖R‖² is summed over the
    // rows in fixed order by the last CTA, so the dynamic row-to-CTA mapping
    // cannot change its rounding.
    block_maxidx(cmax, carg, redv, redi);
    if (tid == 0) {
        P.rrec[blockIdx.x] = RowRecord{0.0, cmax, carg, 0.0};
        __threadfence();
        last = atomicAdd(&st->cnt_r, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    TL_END(2);
    if (!last) return;
    __threadfence();
    double sum = 0.0, mx = -INFINITY;
    long long ax = LLONG_MAX;
    {
        // fixed-order ‖R‖² over r_sq: 16-byte loads, 8 independent accumulators
        // per thread (deep memory-level parallelism for the serial tail)
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const long long T = blockDim.x;
        // a shard's slice of the global r_sq starts at row0, which may be odd:
        // the first row then goes scalar and the rest in aligned pairs
        const int off = (reinterpret_cast<uintptr_t>(P.r_sq) & 15) ? 1 : 0;
        const long long h = (m - off) >> 1;
        const double2* r2 = reinterpret_cast<const double2*>(P.r_sq + off);
        if (off && tid == 0) acc[1] += __ldcg(P.r_sq);
        long long k = tid;
        for (; k + 3 * T < h; k += 4 * T) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 v = __ldcg(r2 + k + u * T);
                acc[2 * u] += v.x;
                acc[2 * u + 1] += v.y;
            }
        }
        for (; k < h; k += T) {
            const double2 v = __ldcg(r2 + k);
            acc[0] += v.x;
            acc[1] += v.y;
        }
        if (((m - off) & 1) && tid == 0) acc[0] += __ldcg(P.r_sq + m - 1);
        sum = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    }
    for (int k = tid; k < (int)gridDim.x; k += blockDim.x) {
        const double* rpp = reinterpret_cast<const double*>(P.rrec + k);
        maxidx_merge(mx, ax, __ldcg(rpp + 1), __ldcg(reinterpret_cast<const long long*>(rpp + 2)));
    }
    sum = block_sum(sum, redv);
    block_maxidx(mx, ax, redv, redi);
    if (tid == 0) {
        st->r_next = 0ull;
        AXB_STAMP(7);
    }
    // the TMA ring is idle now: reuse it as selection scratch
    finalize<UPDATE>(P, st, sum, mx, ax, stage, (long long)S * TW);
    TL_END(2);
}

size_t tma_smem_bytes(const Params& P) {
    return (size_t)P.r_stages * P.r_chunk * 8 * (P.r_zstage ? 2 : 1) + 2 * P.r_stages * 8;
}

// ------------------------------------------------------------------------
// K4 as a TMA ring: y_j = B_j·R_iᵀ over this rank's column slice (and, when G is
// not cached, g_l = A_l·A_iᵀ), with K2's machinery: one producer warp grabs rows
// one at a time from an atomic counter and streams each row in r_chunk-column
// tiles together with the matching tile of the shared vector (R_i or A_i) into
// an r_stages-deep mbarrier ring; eight consumer warps form the dot products
// from shared memory.  Each warp's partial of a row is kept and combined in
// fixed warp order, so the dynamic row-to-CTA mapping cannot change rounding.
// The ring's smem is K2's, so all iteration kernels share one carve-out.
// (The CTA-per-row k_yg ran at ~50% of HBM bandwidth at config 3: 2048 short
// CTAs, each re-reading R_i from L2 with a block barrier per row.)
__global__ void __launch_bounds__(kTmaThreads, 2) k_yg_tma(Params P, int with_g) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ long long stage_row[32];
    __shared__ double rpart[kRowsKept * kTmaConsumerWarps];
    __shared__ long long rowid[kRowsKept];
    __shared__ bool last;
    pdl_wait();
    pdl_trigger();
    DevState* st = P.st;
    if (halted(st)) return;
    TL_BEGIN(0, 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int TW = P.r_chunk;
    const int S = P.r_stages;
    double* stage = reinterpret_cast<double*>(dsm);
    double* vstage = stage + (size_t)S * TW;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(dsm + (size_t)S * TW * 16);
    unsigned long long* empty = full + S;
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kTmaConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const double* Ri;
    const double* Ai;
    if (P.pack) {  // sharded: the owner's row arrived through the allreduce
        Ri = P.pack;
        Ai = P.pack + P.n;
    } else {
        const long long il = st->sel - P.row0;
        Ri = P.R + il * P.n;
        Ai = P.A + il * P.p;
    }
    const long long q = P.q, nrows = q + (with_g ? P.m : 0);
    const long long lenB = P.c1 - P.c0, lenA = P.p;
    if (warp == kTmaConsumerWarps) {
        // ---- producer: one row per grab, tiles of the row and of the vector ----
        int s = 0;
        unsigned round = 0;
        if (lane == 0) {
            for (;;) {
                const long long r = (long long)atomicAdd(&st->yg_next, 1ull);
                if (r >= nrows) break;
                const bool isB = r < q;
                AXB_CHECK(r >= 0 && r < nrows && (isB || P.A));
                const double* src = isB ? P.B + r * P.n + P.c0 : P.A + (r - q) * P.p;
                const double* vec = isB ? Ri + P.c0 : Ai;
                const long long len = isB ? lenB : lenA;
                for (long long c0 = 0; c0 < len; c0 += TW) {
                    if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
                    stage_row[s] = r;
                    const unsigned bytes = (unsigned)(min((long long)TW, len - c0) * 8);
                    mbar_expect_tx(&full[s], 2u * bytes);
                    tma_load_1d(stage + (size_t)s * TW, src + c0, bytes, &full[s]);
                    tma_load_1d(vstage + (size_t)s * TW, vec + c0, bytes, &full[s]);
                    if (++s == S) {
                        s = 0;
                        ++round;
                    }
                }
            }
            if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
            stage_row[s] = -1;  // sentinel: no bytes
            mbar_arrive(&full[s]);
        }
    } else {
        // ---- 8 consumer warps ----
        int s = 0, nkeep = 0;
        unsigned round = 0;
        auto flush = [&](int nk) {
            asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumerWarps * 32) : "memory");
            for (int t = tid; t < nk; t += kTmaConsumerWarps * 32) {
                double a = 0.0;
                for (int w = 0; w < kTmaConsumerWarps; ++w) a += rpart[t * kTmaConsumerWarps + w];
                const long long r = rowid[t];
                AXB_CHECK(r >= 0 && r < nrows);
                if (r < q) P.y[r] = a;
                else P.g[r - q] = a;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumerWarps * 32) : "memory");
        };
        for (;;) {
            mbar_wait(&full[s], round & 1);
            const long long row = stage_row[s];
            if (row < 0) break;
            const long long len = row < q ? lenB : lenA;
            double acc = 0.0;
            for (long long c0 = 0; c0 < len; c0 += TW) {
                if (c0 > 0) mbar_wait(&full[s], round & 1);
                const int h = (int)(min((long long)TW, len - c0) >> 1);
                const double2* b2 = reinterpret_cast<const double2*>(stage + (size_t)s * TW);
                const double2* v2 = reinterpret_cast<const double2*>(vstage + (size_t)s * TW);
#pragma unroll 4
                for (int k = tid; k < h; k += kTmaConsumerWarps * 32) {
                    const double2 b = b2[k], v = v2[k];
                    acc += b.x * v.x;
                    acc += b.y * v.y;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (++s == S) {
                    s = 0;
                    ++round;
                }
            }
            acc = warp_sum(acc);
            if (lane == 0) rpart[nkeep * kTmaConsumerWarps + warp] = acc;
            if (tid == 0) rowid[nkeep] = row;
            if (++nkeep == kRowsKept) {
                flush(nkeep);
                nkeep = 0;
            }
        }
        flush(nkeep);
    }
    // the last CTA out resets the row counter for the next launch
    __syncthreads();
    TL_END(0);
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(&st->cnt_yg, 1u) == gridDim.x - 1;
        if (last) {
            st->yg_next = 0ull;
            st->cnt_yg = 0u;
        }
    }
}

// ------------------------------------------------------------------------
// Sharded selection (after ONE grouped allgather of every shard's ‖R_l‖² slice
// into the global r_sq_g and of the per-shard records).  Every rank then holds
// the global ‖R_l‖² and ‖A_l‖², so every rank runs the single-GPU selection over
// the GLOBAL rows — membership, ordered member-mass prefix, one xoshiro draw, the
// two-level search, the tie guard and the reference's sequential walk as the
// exact fallback (solver.hpp:241-254, rng.hpp:84-99) — on identical inputs with
// an identical RNG state, and all ranks agree on the row bit for bit with no
// further exchange.  (The first version exchanged per-shard member masses and let
// the owner search alone; it could not replay the reference's sequential walk
// on a near-tie because no rank saw all rows.)
//
//   mode 0  norms pass: commit ‖R‖², max ratio / argmax, ‖X−X_ref‖², no selection
//   mode 1  iteration: commit, trace, stop / divergence logic, select the next row
//   mode 2  select only, from the committed state (ensure_selection)
//
// The O(m_global) membership pass is spread over sel1_grid CTAs (a group's sum does
// not depend on which CTA forms it); the last CTA to arrive commits and selects.
__global__ void __launch_bounds__(kThreads) k_sel1(Params P, int mode) {
    __shared__ SelShared sh;
    __shared__ bool last;
    __shared__ long long s_sel;
    __shared__ int s_err;
    pdl_wait();
    DevState* st = P.st;
    if (mode == 1 && halted(st)) return;
    const int tid = threadIdx.x;
    const int fmode = mode == 1 ? st->fin_mode : FIN_NORMS;
    const long long mg = P.m_global;
    double s = 0.0, err = 0.0, mx = -INFINITY;
    long long ax = LLONG_MAX;
    if (mode == 2) {
        s = st->r_fro_sq;
        mx = st->max_ratio;
        ax = st->argmax;
    } else {
        for (int r = 0; r < P.world; ++r) {
            const double* rec = P.recs + 4 * r;
            s += rec[0];
            maxidx_merge(mx, ax, rec[1], (long long)rec[2]);
            err += rec[3];
        }
    }
    const bool diverged = fmode != FIN_NORMS && !isfinite(s);  // solver.hpp:306-307
    const bool greedy = P.method == 2 || P.method == 3;
    const bool masses = mode != 0 && greedy && !st->replay && s > 0.0 && !diverged &&
                        st->status != ST_ERROR;
    Member mem;
    mem.a_sq = P.a_sq_g;
    mem.r_sq = P.r_sq_g;
    mem.smem = 0;
    mem.row0 = 0;
    mem.argmax = ax;
    mem.r_fro = s;
    mem.zeta = __dadd_rn(__dmul_rn(P.theta, __ddiv_rn(mx, s)),
                         __ddiv_rn(__dsub_rn(1.0, P.theta), P.a_fro_sq));  // as make_member
    if (masses) {
        const long long ng = (mg + 31) / 32;
        const long long per = (ng + gridDim.x - 1) / gridDim.x;
        const long long gb = (long long)blockIdx.x * per;
        grbk_group_sums(mem, mg, P.gsum, min(ng, gb), min(ng, gb + per));
    }
    __threadfence();  // this CTA's group sums before its arrival
    __syncthreads();
    if (tid == 0) last = gridDim.x == 1 || atomicAdd(&st->cnt_sel1, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0) {
        st->cnt_sel1 = 0u;
        if (mode != 2) {
            st->err_sq = err;
            st->r_fro_sq = s;
            st->max_ratio = mx;
            st->argmax = ax;
            st->sel_valid = 0;
            const double cf = P.c_fro > 0.0 ? P.c_fro : 1.0;
            const double rel = sqrt(s > 0.0 ? s : 0.0) / cf;
            if (diverged) {
                st->status = ST_ERROR;
                st->err_code = 4;
                st->err_k = st->k;
                st->err_val = sqrt(fabs(s));
            } else if (mode == 1 && fmode == FIN_ITERATION) {
                const unsigned long long k = st->k;
                const double metric = P.stop_kind == 0 ? err / P.ref_sq : rel;
                const unsigned long long slot = k - st->k0;
                if (slot < P.trace_cap) {
                    P.trace_row[slot] = (long long)P.pack[P.n + P.p];
                    P.trace_metric[slot] = metric;
                    P.trace_rel[slot] = rel;
                }
                st->k = k + 1;
                st->metric = metric;
                if (st->run_mode && metric <= P.tol) st->status = ST_PAUSE;
                else if (st->run_mode && !(s > 0.0)) st->status = ST_ZERO;
            } else {
                st->metric = P.stop_kind == 0 ? err / P.ref_sq : rel;
            }
        }
    }
    __syncthreads();
    if (mode == 0) return;
    if (st->status != ST_RUN || st->k >= st->k_limit) return;  // nothing to select
    // ---- the selection, identical on every rank ----
    sel_snapshot(st, sh);  // rollback point (an unused pre-selection is undone)
    if (tid == 0) {
        s_sel = -1;
        s_err = 0;
    }
    __syncthreads();
    if (greedy && !st->replay) {
        long long row = -1;
        int e = 2;  // "greedy threshold: zero residual" (solver.hpp:213-214)
        if (s > 0.0) e = grbk_pick(P, st, mem, P.gsum, mg, 0, &row, sh);
        if (tid == 0) {
            s_sel = row;
            s_err = e;
        }
    } else if (tid == 0) {
        const int method = P.method;
        if (st->replay) {
            const long long row = P.forced_rows[st->k - st->k0];
            if (row < 0 || row >= mg || !(P.a_sq_g[row] > 0.0)) s_err = 2;
            else s_sel = row;
            if (method == 1 || method == 2 || method == 3) (void)rng_next(st->rng);
            if (method == 0 && !s_err) st->cyclic_pos = (unsigned long long)((row + 1) % mg);
        } else if (method == 4) {  // MWRBK: smallest global argmax (solver.hpp:258)
            if (st->argmax == LLONG_MAX) s_err = 2;
            else s_sel = st->argmax;
        } else if (method == 0) {  // BK over the global rows (solver.hpp:197-206)
            s_err = 2;
            for (long long tries = 0; tries < mg; ++tries) {
                const long long i = (long long)st->cyclic_pos;
                st->cyclic_pos = (st->cyclic_pos + 1) % (unsigned long long)mg;
                if (P.a_sq_g[i] > 0.0) {
                    s_sel = i;
                    s_err = 0;
                    break;
                }
                ++st->skipped_zero_rows;
            }
        } else {  // RBK on the global CDF (solver.hpp:209, rng.hpp:84-99)
            const double* cum = P.rbk_cum;
            const double total = cum[mg - 1];
            if (!(total > 0.0)) {
                s_err = 2;
            } else {
                const double target = __dmul_rn(rng_unit(st->rng), total);
                long long lo = 0, hi = mg - 1;
                while (lo < hi) {
                    const long long mid = (lo + hi) / 2;
                    if (cum[mid] <= target) lo = mid + 1;
                    else hi = mid;
                }
                while (lo > 0 && cum[lo] == cum[lo - 1]) --lo;
                s_sel = lo;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (s_err) {
            st->status = ST_ERROR;
            st->err_code = s_err;
            st->err_k = st->k;
            st->sel_valid = 0;
        } else {
            // the pack itself is k_pack's (many CTAs): the owner copies its row,
            // the previous owner clears its stale one
            AXB_CHECK(s_sel >= 0 && s_sel < mg);
            st->sel = s_sel;
            st->sel_valid = 1;
            st->pack_prev = st->packed;
            st->packed = (s_sel / P.m) == P.rank ? 1 : 0;  // equal contiguous shards
        }
    }
}

// Sharded selection, part 3: R_i | A_i | i | coef into pack_send on the owning
// rank (zeros where this rank packed the previous row), across pack_grid CTAs.
// The copy had run in the selection kernel's single CTA as one dependent load→store chain per
// thread: ~80 µs per iteration on the owner at the world-8 shard of config 5.
__global__ void __launch_bounds__(kThreads) k_pack(Params P) {
    pdl_wait();
    pdl_trigger();
    const DevState* st = P.st;
    if (st->status != ST_RUN || st->k >= st->k_limit) return;  // k_sel1 did not select
    const bool mine = st->packed != 0, was = st->pack_prev != 0;
    if (!mine && !was) return;
    const long long n = P.n, p = P.p;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double* __restrict__ out = P.pack_send;
    if (mine) {
        const long long il = st->sel - P.row0;
        AXB_CHECK(il >= 0 && il < P.m);
        const double* __restrict__ Rr = P.R + il * n;
        const double* __restrict__ Ar = P.A + il * p;
        for (long long k = t0; k < n; k += stride) out[k] = __ldcg(Rr + k);
        for (long long k = t0; k < p; k += stride) out[n + k] = __ldg(Ar + k);
        if (t0 == 0) {
            out[n + p] = (double)st->sel;
            out[n + p + 1] = __ddiv_rn(P.alpha, P.a_sq[il]);
        }
    } else {
        for (long long k = t0; k < n + p + 2; k += stride) out[k] = 0.0;
    }
}

// ------------------------------------------------------------------------
// Small systems (everything L2-resident, per-iteration work ≪ launch latency):
// ONE persistent cooperative kernel runs a whole batch.  Per iteration:
//   y (+g) phase ─grid.sync─ z + X phase ─grid.sync─ R update + records ─grid.sync─
//   every CTA reduces the records (fixed order) and selects the next row in its
//   own shared-memory copy of DevState (same xoshiro stream, same inputs →
//   identical results), so no fourth barrier is needed; CTA 0 writes the trace
//   and, at the end, the state.
// ------------------------------------------------------------------------
// K3 split: the greedy pre-selection of the next row across sel_grid CTAs.
// K2's last CTA publishes ‖R‖², max ratio and argmax and sets sel_pending; here
// every CTA forms the member-mass sums of its slice of the 32-row groups and
// the last CTA to finish runs the ordered prefix, the draw and the search —
// the same arithmetic as the single-CTA path (grbk_group_sums / grbk_pick),
// with the O(m) membership pass spread over the SMs.
__global__ void __launch_bounds__(kThreads) k_sel_greedy(Params P) {
    __shared__ SelShared sh;
    __shared__ bool last;
    // K4 (next in the stream) waits for this grid, which waits for K2, so letting
    // it launch early is safe; it then prefetches B while K2 drains
    if (P.sel_early) pdl_trigger();
    pdl_wait();
    pdl_trigger();
    DevState* st = P.st;
    if (!st->sel_pending) return;
    TL_BEGIN(3, 1);
    const long long m = P.m, ng = (m + 31) / 32;
    const bool live = st->r_fro_sq > 0.0;
    if (live) {
        const Member mem = make_member(P, st, P.theta);
        const long long per = (ng + gridDim.x - 1) / gridDim.x;
        const long long gb = (long long)blockIdx.x * per;
        grbk_group_sums(mem, m, P.gsum, gb, min(ng, gb + per));
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&st->cnt_sel, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    TL_END(3);
    if (!last) return;
    __threadfence();
    sel_snapshot(st, sh);
    long long row = 0;
    int err = 2;  // "greedy threshold: zero residual"
    if (live) {
        const Member mem = make_member(P, st, P.theta);
        err = grbk_pick(P, st, mem, P.gsum, P.m, P.row0, &row, sh);
    }
    __syncthreads();
    sel_commit(P, st, err, row);
    if (threadIdx.x == 0) {
        st->sel_pending = 0;
        st->cnt_sel = 0u;
    }
    TL_END(3);
}

constexpr int kPersistThreads = 256;

// Execution groups of the persistent iteration: a cooperative grid working on
// one system (k_persist), or one CTA owning a whole small system
// (k_persist_batch, SURVEY §8 F3 — many independent solves in one launch).
struct GridGroup {
    static constexpr bool kWholeChip = true;  // one system on the cooperative grid
    cooperative_groups::grid_group g;
    __device__ int rank() const { return (int)blockIdx.x; }
    __device__ int size() const { return (int)gridDim.x; }
    __device__ void sync() { g.sync(); }
};
struct SoloGroup {
    static constexpr bool kWholeChip = false;  // one CTA per system (k_persist_batch)
    __device__ int rank() const { return 0; }
    __device__ int size() const { return 1; }
    __device__ void sync() { __syncthreads(); }
};

// per-phase time of the persistent body (CTA 0, thread 0) into DevState::dbg:
// select, y, z-partials+X, z-combine, R update, finalize, barrier waits, iterations
// (build with -DAXB_TRACE_PERSIST; read with axb_solver_debug_state)
#ifdef AXB_TRACE_PERSIST
#define PT_DECL unsigned long long pt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt_t = 0
#define PT_MARK(slot)                                          \
    do {                                                       \
        if (tid == 0 && grid.rank() == 0) {                    \
            unsigned long long t_;                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
            if ((slot) >= 0 && pt_t) pt_acc[(slot)] += t_ - pt_t; \
            pt_t = t_;                                         \
        }                                                      \
    } while (0)
#define PT_ITER() (pt_acc[7] += (tid == 0 && grid.rank() == 0))
#define PT_STORE()                                                   \
    do {                                                             \
        if (tid == 0 && grid.rank() == 0)                            \
            for (int s_ = 0; s_ < 8; ++s_) P.st->dbg[s_] = pt_acc[s_]; \
    } while (0)
#else
#define PT_DECL
#define PT_MARK(slot) ((void)0)
#define PT_ITER() ((void)0)
#define PT_STORE() ((void)0)
#endif

template <class Grp, int kT>
__device__ __forceinline__ void persist_body(const Params& P, Grp grid) {
    PT_DECL;
    constexpr int kW = kT / 32;
    constexpr int kSub = kT / kPersistThreads;  // 256-thread sub-blocks (z items)
    extern __shared__ double pscratch[];  // selection scratch: ⌈m/32⌉ group sums
    __shared__ DevState lst;
    __shared__ SelShared sh;
    __shared__ double red[32];
    __shared__ long long redi[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = P.m, n = P.n, p = P.p, q = P.q;
    const long long gw = (long long)grid.rank() * kW + warp;  // global warp
    const long long nw = (long long)grid.size() * kW;
    long long g_prev = -1;  // CSR A: the Gram row scattered into g last (CTA 0)
    if (tid == 0) lst = *P.st;
    __syncthreads();
    for (;;) {
        if (lst.status != ST_RUN || lst.k >= lst.k_limit) break;
        PT_MARK(-1);
        PT_ITER();
        // K3 (every CTA, identically); update_row(i) brings its own row (k_set_sel)
        if (!lst.sel_valid && lst.fin_mode != FIN_UPDATE_ROW) {
            long long row = 0;
            if (tid == 0) sh.err = 0;
            __syncthreads();
            const int err = select_rows(P, &lst, P.method, P.theta, &row, sh, pscratch,
                                        (m + 31) / 32);
            __syncthreads();
            if (tid == 0) {
                if (err) {
                    lst.status = ST_ERROR;
                    lst.err_code = err;
                    lst.err_k = lst.k;
                } else {
                    AXB_CHECK(row >= 0 && row < m);
                    lst.sel = row;
                    lst.coef = __ddiv_rn(P.alpha, P.a_sq[row]);
                    lst.sel_valid = 1;
                }
            }
            __syncthreads();
            if (lst.status != ST_RUN) break;
        }
        PT_MARK(0);
        const long long sel = lst.sel;
        const double coef = lst.coef;
        const double* Ri = P.R + sel * n;
        const double* Ai = P.A + sel * p;
        // ---- y = B·R_iᵀ (+ g = A·A_iᵀ) ----
        // two rows per warp pass sharing the vector loads (y rows, then g rows)
        if (P.b_rp) {
            // CSR B: y_j = Σ over B_j's stored entries of B_jk·R_ik (matvec_into,
            // solver.hpp:489-492), a warp per row
            const long long* const brp = P.b_rp;
            const int* const bci = P.b_ci;
            const double* const bv = P.b_v;
            for (long long j = gw; j < q; j += nw) {
                double a = 0.0;
                for (long long e = brp[j] + lane; e < brp[j + 1]; e += 32) {
                    AXB_CHECK(bci[e] >= 0 && bci[e] < n);
                    a += __ldg(bv + e) * __ldcg(Ri + __ldg(bci + e));
                }
                a = warp_sum(a);
                if (lane == 0) P.y[j] = a;
            }
        }
        if (P.g_rp) {
            // CSR A: the Gram row G_i (CSR, formed once in the reference's order)
            // scattered into the dense coefficient vector g, whose other entries stay
            // exactly zero, so the R phase below touches only l ∈ nz(G_i)
            // (solver.hpp:294-295).  CTA 0 clears the previous row's entries first;
            // the grid barrier publishes g before the R phase reads it.
            if (grid.rank() == 0) {
                double* const go = P.g;
                if (g_prev >= 0)
                    for (long long e = P.g_rp[g_prev] + tid; e < P.g_rp[g_prev + 1]; e += kT)
                        go[P.g_ci[e]] = 0.0;
                __syncthreads();
                AXB_CHECK(sel >= 0 && sel < m);
                for (long long e = P.g_rp[sel] + tid; e < P.g_rp[sel + 1]; e += kT) {
                    AXB_CHECK(P.g_ci[e] >= 0 && P.g_ci[e] < m);
                    go[P.g_ci[e]] = P.g_v[e];
                }
                g_prev = sel;
            }
        }
        if (!P.b_rp || (!P.G && !P.g_rp)) {
            double* const yo = P.y;
            double* const go = P.g;
            const double* const Bb = P.B;
            const double* const Ab = P.A;
            if (Grp::kWholeChip && q <= nw && !P.b_rp) {
                // fewer rows than warps (config 2: 400 rows, 1184 warps): one row per
                // warp, 6 loads per lane in flight — a 2000-column row is 6 L2 round
                // trips instead of 8.  (8 in flight, or the pair form, spill: the body is
                // at 243 registers, and config 2 dropped from 35.3k to 28.6k it/s.)
                if (gw < q) {
                    const double a0 = warp_dot_u<6>(Bb + gw * n, Ri, n, lane, (n & 1) == 0, true);
                    if (lane == 0) yo[gw] = a0;
                }
            } else
            for (long long it = gw; it < q && !P.b_rp; it += 2 * nw) {
                const long long it1 = it + nw;
                double a0, a1;
                warp_dot_pair(Bb + it * n, it1 < q ? Bb + it1 * n : nullptr, Ri, n, lane,
                              (n & 1) == 0, true, a0, a1);
                if (lane == 0) {
                    yo[it] = a0;
                    if (it1 < q) yo[it1] = a1;
                }
            }
            if (!P.G && !P.g_rp) {
                for (long long it = gw; it < m; it += 2 * nw) {
                    const long long it1 = it + nw;
                    double a0, a1;
                    warp_dot_pair(Ab + it * p, it1 < m ? Ab + it1 * p : nullptr, Ai, p, lane,
                                  (p & 1) == 0, false, a0, a1);
                    if (lane == 0) {
                        go[it] = a0;
                        if (it1 < m) go[it1] = a1;
                    }
                }
            }
        }
        PT_MARK(1);
        grid.sync();
        PT_MARK(6);
        // ---- z = yᵀ·B, stage 1: (column slab × row chunk) partials; X update ----
        if (P.bt_rp) {
            // CSR B: z_c = Σ over column c of B (the rows of Bᵀ, ascending j) of
            // y_j·B_jc, a warp per column, written straight to z
            const long long* const trp = P.bt_rp;
            const int* const tci = P.bt_ci;
            const double* const tv = P.bt_v;
            for (long long c = gw; c < n; c += nw) {
                double a = 0.0;
                for (long long e = trp[c] + lane; e < trp[c + 1]; e += 32) {
                    AXB_CHECK(tci[e] >= 0 && tci[e] < q);
                    a += __ldcg(P.y + __ldg(tci + e)) * __ldg(tv + e);
                }
                a = warp_sum(a);
                if (lane == 0) P.z[c] = a;
            }
        } else {
            const int items = P.z_nslab * P.z_nj;
            const int sub = tid / kPersistThreads, stid = tid % kPersistThreads;
            for (int itm = grid.rank() * kSub + sub; itm < items; itm += grid.size() * kSub) {
                const int slab = itm % P.z_nslab, jc = itm / P.z_nslab;
                const long long j0 = (long long)jc * P.z_jrows, j1 = min(q, j0 + P.z_jrows);
                const long long c = (long long)slab * (2 * kPersistThreads) + 2 * stid;
                double a0 = 0.0, a1 = 0.0;
                if (c < n) {
#pragma unroll 8
                    for (long long j = j0; j < j1; ++j) {
                        const double yj = __ldcg(P.y + j);
                        a0 += yj * __ldg(P.B + j * n + c);
                        if (c + 1 < n) a1 += yj * __ldg(P.B + j * n + c + 1);
                    }
                    double* zp = P.zpart + (long long)jc * n;
                    zp[c] = a0;
                    if (c + 1 < n) zp[c + 1] = a1;
                }
            }
        }
        double xacc = 0.0;
        const double* const yb = P.y;
        double* const Xb = P.X;
        const double* const Xrefb = P.Xref;
        if (P.a_rp) {
            // CSR A: X_t += (coef·A_it)·y for t ∈ nz(A_i) only, and the reference's
            // incremental ‖X−X_ref‖² tracker, Σ_j (d1² − d0²) per updated row
            // (solver.hpp:272-289); a warp per (stored entry, 256-column segment),
            // so a 15-entry row of a 1024-column X keeps 60 warps busy for one
            // L2 round trip each instead of 15 warps for 32 dependent ones
            const long long e0 = P.a_rp[sel], e1 = P.a_rp[sel + 1];
            const long long nseg = (q + 32 * kXS - 1) / (32 * kXS);
            for (long long it = gw; it < (e1 - e0) * nseg; it += nw) {
                const long long e = e0 + it / nseg;
                const long long t = P.a_ci[e];
                AXB_CHECK(t >= 0 && t < p);
                const double f = __dmul_rn(coef, P.a_v[e]);
                // inlined on the cooperative grid; behind a call in the batched kernel,
                // which runs at a 128-register cap
                if constexpr (Grp::kWholeChip)
                    xacc += x_segment_inc(Xb + t * q, Xrefb ? Xrefb + t * q : nullptr, yb, q,
                                          it % nseg, f, lane);
                else
                    xacc += x_segment_inc_call(Xb + t * q, Xrefb ? Xrefb + t * q : nullptr, yb, q,
                                               it % nseg, f, lane);
            }
        }
        for (long long t = gw; t < p && !P.a_rp; t += nw) {
            const double f = __dmul_rn(coef, Ai[t]);
            if (f == 0.0 && !Xrefb) continue;  // A_it = 0: X_t unchanged (solver.hpp:272-273)
            double* xr = Xb + t * q;
            const double* rr = Xrefb ? Xrefb + t * q : nullptr;
            for (long long k0 = lane; k0 < q; k0 += 32 * 4) {
                double xv[4], yv[4], rv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const long long k = k0 + 32 * u;
                    if (k < q) {
                        xv[u] = xr[k];
                        yv[u] = __ldcg(yb + k);
                        rv[u] = rr ? rr[k] : 0.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const long long k = k0 + 32 * u;
                    if (k < q) {
                        const double x1 = __dadd_rn(xv[u], __dmul_rn(f, yv[u]));
                        xr[k] = x1;
                        if (rr) {
                            const double d1 = x1 - rv[u];
                            xacc += d1 * d1;
                        }
                    }
                }
            }
        }
        xacc = block_sum(xacc, red);
        if (tid == 0) P.xpart[grid.rank()] = xacc;
        PT_MARK(2);
        grid.sync();
        PT_MARK(6);
        // ---- z stage 2: fixed-order combine of the row-chunk partials ----
        for (long long c = (long long)grid.rank() * kT + tid; c < n && !P.bt_rp;
             c += (long long)grid.size() * kT) {
            double a = 0.0;
            for (int k = 0; k < P.z_nj; ++k) a += __ldcg(P.zpart + (long long)k * n + c);
            P.z[c] = a;
        }
        PT_MARK(3);
        grid.sync();
        PT_MARK(6);
        // ---- R update + row norms (warp per row, static mapping) ----
        // Pointers are hoisted into registers: P may live in shared memory
        // (k_persist_batch) and a generic store could alias it otherwise.
        double wsum = 0.0, wmax = -INFINITY;
        long long warg = LLONG_MAX;
        double* const Rb = P.R;
        const double* const zb = P.z;
        const double* const Gsel = P.G ? P.G + sel * m : nullptr;
        const double* const gv = P.g;
        double* const rsq = P.r_sq;
        const double* const asq = P.a_sq;
        auto coef_of = [&](long long l) { return Gsel ? __ldcg(Gsel + l) : __ldcg(gv + l); };
        auto record = [&](long long l, double rs) {
            wsum += rs;
            const double as = asq[l];
            if (as > 0.0) maxidx_merge(wmax, warg, __ddiv_rn(rs, as), l);
        };
        if ((n & 1) == 0) {
            // two rows per warp pass (l, l + nw — the warp's own next row), 16-byte
            // accesses, 4 segments per lane in flight: 12 loads outstanding per lane
            const long long h = n >> 1;
            const double2* z2 = reinterpret_cast<const double2*>(zb);
            // the Gram coefficients of the warp's next 32 rows are fetched in one
            // round trip (lane j holds row gw + (t0 + j)·nw) and shuffled out
            double gpre = 0.0;
            long long t = 0;  // index of l0 among the warp's rows
            for (long long l0 = gw; l0 < m; l0 += 2 * nw, t += 2) {
                if ((t & 31) == 0) {
                    const long long lr = gw + (t + lane) * nw;
                    gpre = lr < m ? coef_of(lr) : 0.0;
                }
                const long long l1 = l0 + nw;
                const bool has1 = l1 < m;
                const double g0 = __shfl_sync(0xffffffffu, gpre, (int)(t & 31));
                const double g1v = __shfl_sync(0xffffffffu, gpre, (int)((t + 1) & 31));
                const double g1 = has1 ? g1v : 0.0;
                const bool up0 = g0 != 0.0, up1 = g1 != 0.0;  // sparse-G skip (:294-295)
                const double f0 = __dmul_rn(coef, g0), f1 = __dmul_rn(coef, g1);
                double2* row0 = reinterpret_cast<double2*>(Rb + l0 * n);
                double2* row1 = reinterpret_cast<double2*>(Rb + (has1 ? l1 : l0) * n);
                double acc0 = 0.0, acc1 = 0.0;
                if (up0 || up1) {
                    for (long long k0 = lane; k0 < h; k0 += 32 * 4) {
                        double2 zv[4], r0[4], r1[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < h) {
                                zv[u] = __ldcg(z2 + k);
                                if (up0) r0[u] = row0[k];
                                if (up1) r1[u] = row1[k];
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < h) {
                                if (up0) {
                                    double2 r;
                                    r.x = __dsub_rn(r0[u].x, __dmul_rn(f0, zv[u].x));
                                    r.y = __dsub_rn(r0[u].y, __dmul_rn(f0, zv[u].y));
                                    row0[k] = r;
                                    acc0 += r.x * r.x;
                                    acc0 += r.y * r.y;
                                }
                                if (up1) {
                                    double2 r;
                                    r.x = __dsub_rn(r1[u].x, __dmul_rn(f1, zv[u].x));
                                    r.y = __dsub_rn(r1[u].y, __dmul_rn(f1, zv[u].y));
                                    row1[k] = r;
                                    acc1 += r.x * r.x;
                                    acc1 += r.y * r.y;
                                }
                            }
                        }
                    }
                }
                double rs0, rs1 = 0.0;
                if (up0) {
                    rs0 = warp_sum(acc0);
                    if (lane == 0) rsq[l0] = rs0;
                } else {
                    rs0 = __ldcg(rsq + l0);
                }
                if (has1) {
                    if (up1) {
                        rs1 = warp_sum(acc1);
                        if (lane == 0) rsq[l1] = rs1;
                    } else {
                        rs1 = __ldcg(rsq + l1);
                    }
                }
                record(l0, rs0);
                if (has1) record(l1, rs1);
            }
        } else {
            for (long long l = gw; l < m; l += nw) {
                const double gl = coef_of(l);
                double rs;
                if (gl == 0.0) {  // R_l unchanged (sparse-G semantics, solver.hpp:294-295)
                    rs = __ldcg(rsq + l);
                } else {
                    const double f = __dmul_rn(coef, gl);
                    double* row = Rb + l * n;
                    double acc = 0.0;
                    for (long long k0 = lane; k0 < n; k0 += 32 * 4) {
                        double rv[4], zv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < n) {
                                rv[u] = row[k];
                                zv[u] = __ldcg(zb + k);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < n) {
                                const double r = __dsub_rn(rv[u], __dmul_rn(f, zv[u]));
                                row[k] = r;
                                acc += r * r;
                            }
                        }
                    }
                    rs = warp_sum(acc);
                    if (lane == 0) rsq[l] = rs;
                }
                record(l, rs);
            }
        }
        // per-CTA record: warp partials combined in warp order (fixed mapping)
        __syncthreads();
        if (lane == 0) {
            red[warp] = wsum;
            sh.scan[warp] = wmax;
            redi[warp] = warg;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, mx = -INFINITY;
            long long ax = LLONG_MAX;
            for (int w = 0; w < kW; ++w) {
                a += red[w];
                maxidx_merge(mx, ax, sh.scan[w], redi[w]);
            }
            P.rrec[grid.rank()] = RowRecord{a, mx, ax, 0.0};
        }
        PT_MARK(4);
        grid.sync();
        PT_MARK(6);
        // ---- every CTA: reduce the records + the ‖X−X_ref‖² partials (block-
        // parallel loads, fixed-order trees → identical in every CTA), finalize ----
        {
            double ps = 0.0, pe = 0.0, pm = -INFINITY;
            long long pa = LLONG_MAX;
            for (int b = tid; b < grid.size(); b += kT) {
                const double* rp = reinterpret_cast<const double*>(P.rrec + b);
                ps += __ldcg(rp);
                maxidx_merge(pm, pa, __ldcg(rp + 1), __ldcg(reinterpret_cast<const long long*>(rp + 2)));
                pe += __ldcg(P.xpart + b);
            }
            ps = block_sum(ps, red);
            pe = block_sum(pe, red);
            block_maxidx(pm, pa, sh.redv, sh.redi);
            if (tid == 0) {
                sh.scan[0] = ps;
                sh.scan[1] = pe;
                sh.scan[2] = pm;
                sh.cand = pa;
            }
            __syncthreads();
        }
        if (tid == 0) {
            const double s = sh.scan[0], mx = sh.scan[2];
            // CSR A: the incremental tracker (clamped at 0, solver.hpp:290); dense: fresh
            double e = sh.scan[1];
            if (P.a_rp) {
                e = __dadd_rn(lst.err_sq, e);
                if (e < 0.0) e = 0.0;
            }
            const long long ax = sh.cand;
            lst.r_fro_sq = s;
            lst.max_ratio = mx;
            lst.argmax = ax;
            lst.err_sq = e;
            lst.sel_valid = 0;
            const double cf = P.c_fro > 0.0 ? P.c_fro : 1.0;
            const double rel = sqrt(s > 0.0 ? s : 0.0) / cf;
            if (!isfinite(s)) {  // solver.hpp:306-307
                lst.status = ST_ERROR;
                lst.err_code = 4;
                lst.err_k = lst.k;
                lst.err_val = sqrt(fabs(s));
            } else if (lst.fin_mode == FIN_UPDATE_ROW) {
                // public update_row(i): no k++, no trace, no stop check; one pass
                lst.metric = P.stop_kind == 0 ? e / P.ref_sq : rel;
                lst.k_limit = lst.k;
            } else {
                const unsigned long long k = lst.k;
                const double metric = P.stop_kind == 0 ? e / P.ref_sq : rel;
                const unsigned long long slot = k - lst.k0;
                AXB_CHECK(k >= lst.k0);
                if (grid.rank() == 0 && slot < P.trace_cap) {
                    P.trace_row[slot] = sel;
                    P.trace_metric[slot] = metric;
                    P.trace_rel[slot] = rel;
                }
                lst.k = k + 1;
                lst.metric = metric;
                if (lst.run_mode && metric <= P.tol) lst.status = ST_PAUSE;
                else if (lst.run_mode && !(s > 0.0)) lst.status = ST_ZERO;
            }
        }
        __syncthreads();
        PT_MARK(5);
        // no barrier needed before the next y phase: it only reads R/B (last
        // written before the grid.sync above) and writes y, which nobody reads
        // until after the next grid.sync
    }
    if (P.g_rp && grid.rank() == 0 && g_prev >= 0) {  // leave g all-zero for the next launch
        for (long long e = P.g_rp[g_prev] + tid; e < P.g_rp[g_prev + 1]; e += kT) P.g[P.g_ci[e]] = 0.0;
    }
    if (grid.rank() == 0 && tid == 0) *P.st = lst;
    PT_STORE();
}

__global__ void __launch_bounds__(kPersistThreads) k_persist(Params P) {
    persist_body<GridGroup, kPersistThreads>(P, GridGroup{cooperative_groups::this_grid()});
}

// One CTA per system: Ps[blockIdx.x] describes an independent solve (its own
// buffers and DevState).  Grid barriers become CTA barriers.
// 512 threads: one CTA must carry a whole system's memory parallelism
// (AXB_BATCH_THREADS=256 / 1024 select the 256-thread, two-per-SM or the
// 1024-thread variant for sweeps)
constexpr int kBatchThreads = 512;
template <int kT>
__global__ void __launch_bounds__(kT, kT <= 256 ? 2 : 1) k_persist_batch(const Params* __restrict__ Ps) {
    __shared__ Params sp;
    if (threadIdx.x == 0) sp = Ps[blockIdx.x];
    __syncthreads();
    persist_body<SoloGroup, kT>(sp, SoloGroup{});
}

// ------------------------------------------------------------------------
// Latency body for small systems (m ≤ kPersistLatRows, BᵀB cached).  A tiny
// system's iteration is a chain of L2 round trips and barriers, not bytes, so
// this body minimises both:
//   * the selection state (r_sq, a_sq, the RBK CDF, the greedy group sums)
//     lives in shared memory; every CTA refreshes r_sq with one batched L2
//     pass per iteration, reduces ‖R‖², max/argmax and ‖X−X_ref‖² from it in a
//     fixed order (identical in every CTA), and selects from shared memory;
//   * z = BᵀB·R_iᵀ with the cached n×n BᵀB — the reference's own formula
//     (solver.hpp:172, :293) — so y and z are both dots with R_i and share one
//     phase, and an iteration needs two grid barriers:
//         [select] y, z (, g) ─sync─ R update ∥ X update ─sync─ [reduce]
//   * loads are issued 8 per lane ahead of the arithmetic (one round trip per
//     row at config-1 widths); X rows go to the last warps, R rows to the first.
// ------------------------------------------------------------------------
__host__ __device__ __forceinline__ size_t persist_lat_smem_doubles(long long m, int) {
    return (size_t)((m + 31) / 32) + 3 * (size_t)m;
}

template <class Grp, int kT>
__device__ __forceinline__ void persist_body_lat(const Params& P, Grp grid) {
    PT_DECL;
    constexpr int kW = kT / 32;
    // loads in flight per lane in the dots (kU) and the row updates (kR; R-row pairs
    // are 3 streams per lane).  The body sits at the 255-register cap, and the spills
    // cost more than deeper batches gain: kU 8 → 4 took the spill stores from 424
    // to 128 bytes and config 1 from 13.7 to 12.5 µs per iteration, a config-4
    // channel from 20.3 to 18.1 µs (tools/sweep_lat_batch.sh; 5 and 6 are worse
    // than both, kR 2, 3 and 6 worse than 4).  -DAXB_LAT_KU / -DAXB_LAT_KR override.
#ifndef AXB_LAT_KU
#define AXB_LAT_KU 4
#endif
#ifndef AXB_LAT_KR
#define AXB_LAT_KR 4
#endif
    constexpr int kU = kT <= 256 ? AXB_LAT_KU : 4;
    constexpr int kR = AXB_LAT_KR;
    extern __shared__ __align__(16) double psm[];
    __shared__ DevState lst;
    __shared__ SelShared sh;
    __shared__ double red[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m = P.m, n = P.n, p = P.p, q = P.q;
    const long long ng = (m + 31) / 32;
    double* const gs = psm;
    double* const rs_s = gs + ng;
    double* const as_s = rs_s + m;
    double* const cum_s = as_s + m;
    const int G = grid.size(), rank = grid.rank();
    const long long gw = (long long)rank * kW + warp;
    const long long nw = (long long)G * kW;
    // pointers hoisted into registers: P may live in shared memory
    const double* const Bb = P.B;
    const double* const BtB = P.BtB;
    const double* const Ab = P.A;
    const double* const Gm = P.G;
    const double* const asq_g = P.a_sq;
    double* const Rb = P.R;
    double* const Xb = P.X;
    const double* const Xrefb = P.Xref;
    double* const yo = P.y;
    double* const zo = P.z;
    double* const go = P.g;
    double* const rsq = P.r_sq;
    double* const xpart = P.xpart;
    const bool vec2 = (n & 1) == 0;
    const int method = P.method;
    if (tid == 0) lst = *P.st;
    for (long long i = tid; i < m; i += kT) {
        as_s[i] = asq_g[i];
        rs_s[i] = __ldcg(rsq + i);
        cum_s[i] = method == 1 ? P.rbk_cum[i] : 0.0;
    }
    __syncthreads();

    // dense A: X items = (row, 32·kR-column segment); CSR A keeps one slot per X row
    const long long x_nseg = (q + 32 * kR - 1) / (32 * kR);
    const long long x_items = p * x_nseg;
    const long long x_slots = P.a_rp ? min(p, nw) : min(x_items, nw);
    // X_t += (coef·A_it)·y (solver.hpp:272-289), warp per row, rows taken from the
    // LAST warps (the R rows start at the first), so a warp rarely does both;
    // each warp's Σ (X − X_ref)² goes to xpart[gw] (fixed slots, fixed order)
    auto x_update = [&](const double* Ai, double coef, long long sel) {
        double xacc = 0.0;
        if (P.a_rp) {
            // CSR A: rows t ∈ nz(A_i) only, incremental Σ_j (d1² − d0²) per row
            // (solver.hpp:272-289), a warp per (stored entry, 256-column segment);
            // the X-owning warps are the last min(p, nw) and each one's slot holds
            // its delta
            const long long w = nw - 1 - gw;
            const long long nx = x_slots;
            const long long e0 = P.a_rp[sel], e1 = P.a_rp[sel + 1];
            const long long nseg = (q + 32 * kXS - 1) / (32 * kXS);
            for (long long it = w; w < nx && it < (e1 - e0) * nseg; it += nx) {
                const long long e = e0 + it / nseg;
                const long long t = P.a_ci[e];
                const double f = __dmul_rn(coef, P.a_v[e]);
                xacc += x_segment_inc_call(Xb + t * q, Xrefb ? Xrefb + t * q : nullptr, yo, q,
                                           it % nseg, f, lane);
            }
            xacc = warp_sum(xacc);
            if (lane == 0 && w < p) xpart[w] = xacc;
            return;
        }
        // items = (row t, segment of 32·kR columns), taken by the warps from the last
        // one down: a long row is spread over several warps, each with ONE batch of
        // loads (a 1024-column row of X was 8 dependent L2 round trips in one warp),
        // and the row's A_it values are fetched lane-parallel first, so rows with
        // A_it = 0 (banded A) cost nothing more
        const long long w = nw - 1 - gw;
        for (long long it0 = w; it0 < x_items; it0 += 32 * nw) {
            const long long itl = it0 + (long long)lane * nw;  // lane j: this warp's j-th item
            const double fl = itl < x_items ? __dmul_rn(coef, Ai[itl / x_nseg]) : 0.0;
            for (int j = 0; j < 32; ++j) {
                const long long it = it0 + (long long)j * nw;
                if (it >= x_items) break;
                const double f = __shfl_sync(0xffffffffu, fl, j);
                if (f == 0.0 && !Xrefb) continue;  // A_it = 0: X_t unchanged (solver.hpp:272-273)
                const long long t = it / x_nseg;
                double* xr = Xb + t * q;
                const double* rr = Xrefb ? Xrefb + t * q : nullptr;
                const long long k0 = (it % x_nseg) * (32 * kR) + lane;
                double xv[kR], yv[kR], rv[kR];
#pragma unroll
                for (int u = 0; u < kR; ++u) {
                    const long long k = k0 + 32 * u;
                    if (k < q) {
                        xv[u] = xr[k];
                        yv[u] = __ldcg(yo + k);
                        rv[u] = rr ? rr[k] : 0.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < kR; ++u) {
                    const long long k = k0 + 32 * u;
                    if (k < q) {
                        const double x1 = __dadd_rn(xv[u], __dmul_rn(f, yv[u]));
                        xr[k] = x1;
                        if (rr) {
                            const double d1 = x1 - rv[u];
                            xacc += d1 * d1;
                        }
                    }
                }
            }
        }
        xacc = warp_sum(xacc);
        // slot = the warp's first X item: only the x_slots X-owning warps write
        if (lane == 0 && w < x_slots) xpart[w] = xacc;
    };

    long long g_prev = -1;  // CSR A: the Gram row scattered into g last (CTA 0)
    for (;;) {
        if (lst.status != ST_RUN || lst.k >= lst.k_limit) break;
        PT_MARK(-1);
        PT_ITER();
        // K3 from shared memory (every CTA, identically); update_row(i) brings its row
        if (!lst.sel_valid && lst.fin_mode != FIN_UPDATE_ROW) {
            long long row = 0;
            if (tid == 0) sh.err = 0;
            __syncthreads();
            const int err = select_rows(P, &lst, method, P.theta, &row, sh, gs, ng, as_s, rs_s,
                                        method == 1 ? cum_s : nullptr);
            __syncthreads();
            if (tid == 0) {
                if (err) {
                    lst.status = ST_ERROR;
                    lst.err_code = err;
                    lst.err_k = lst.k;
                } else {
                    AXB_CHECK(row >= 0 && row < m);
                    lst.sel = row;
                    lst.coef = __ddiv_rn(P.alpha, as_s[row]);
                    lst.sel_valid = 1;
                }
            }
            __syncthreads();
            if (lst.status != ST_RUN) break;
#ifdef AXB_TRACE_PERSIST
            if (tid == 0 && rank == 0 && (method == 2 || method == 3)) {
                unsigned long long t_;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
                pt_acc[3] += t_ - sh.t_groups;
            }
#endif
        }
        PT_MARK(0);
        const long long sel = lst.sel;
        const double coef = lst.coef;
        const double* Ri = Rb + sel * n;
        const double* Ai = Ab + sel * p;
        // ---- phase A: y = B·R_iᵀ and z = BᵀB·R_iᵀ (dots with R_i), g = A·A_iᵀ ----
        if (P.b_rp) {
            // CSR B: y over B's rows and z = BᵀB·R_iᵀ over the CSR BᵀB (formed once in
            // the reference's order, solver.hpp:172, :293), a warp per row
            for (long long it = gw; it < q + n; it += nw) {
                const bool isy = it < q;
                const long long r = isy ? it : it - q;
                const long long* rp = isy ? P.b_rp : P.btb_rp;
                const int* ci = isy ? P.b_ci : P.btb_ci;
                const double* vv = isy ? P.b_v : P.btb_v;
                double a = 0.0;
                for (long long e = rp[r] + lane; e < rp[r + 1]; e += 32) {
                    AXB_CHECK(ci[e] >= 0 && ci[e] < n);
                    a += __ldg(vv + e) * __ldcg(Ri + __ldg(ci + e));
                }
                a = warp_sum(a);
                if (lane == 0) (isy ? yo : zo)[r] = a;
            }
        }
        if (P.g_rp && rank == 0) {
            // CSR A: scatter G_i into g (CTA 0, after clearing the previous row's
            // entries); phase C reads g after the barrier
            if (g_prev >= 0)
                for (long long e = P.g_rp[g_prev] + tid; e < P.g_rp[g_prev + 1]; e += kT)
                    go[P.g_ci[e]] = 0.0;
            __syncthreads();
            for (long long e = P.g_rp[sel] + tid; e < P.g_rp[sel + 1]; e += kT)
                go[P.g_ci[e]] = P.g_v[e];
        }
        if (P.g_rp) g_prev = sel;
        if (!P.b_rp || (!Gm && !P.g_rp)) {
            const long long nd = P.b_rp ? 0 : q + n;
            for (long long it = gw; it < nd; it += 2 * nw) {
                const long long it1 = it + nw;
                const double* r0 = it < q ? Bb + it * n : BtB + (it - q) * n;
                const double* r1 =
                    it1 < nd ? (it1 < q ? Bb + it1 * n : BtB + (it1 - q) * n) : nullptr;
                double a0, a1;
                warp_dot_pair_u<kU>(r0, r1, Ri, n, lane, vec2, true, a0, a1);
                if (lane == 0) {
                    if (it < q) yo[it] = a0;
                    else zo[it - q] = a0;
                    if (r1) {
                        if (it1 < q) yo[it1] = a1;
                        else zo[it1 - q] = a1;
                    }
                }
            }
            if (!Gm && !P.g_rp) {
                for (long long it = gw; it < m; it += 2 * nw) {
                    const long long it1 = it + nw;
                    double a0, a1;
                    warp_dot_pair(Ab + it * p, it1 < m ? Ab + it1 * p : nullptr, Ai, p, lane,
                                  (p & 1) == 0, false, a0, a1);
                    if (lane == 0) {
                        go[it] = a0;
                        if (it1 < m) go[it1] = a1;
                    }
                }
            }
        }
        PT_MARK(1);
        grid.sync();
        PT_MARK(6);
        // ---- phase C: R_l −= (coef·G_il)·z, ‖R_l‖² (solver.hpp:294-305); X ----
        {
            const double* const Gsel = Gm ? Gm + sel * m : nullptr;
            auto coef_of = [&](long long l) { return Gsel ? __ldg(Gsel + l) : __ldcg(go + l); };
            if (vec2) {
                const long long h = n >> 1;
                const double2* z2 = reinterpret_cast<const double2*>(zo);
                for (long long l0 = gw; l0 < m; l0 += 2 * nw) {
                    const long long l1 = l0 + nw;
                    const bool has1 = l1 < m;
                    const double g0 = coef_of(l0);
                    const double g1 = has1 ? coef_of(l1) : 0.0;
                    const bool up0 = g0 != 0.0, up1 = g1 != 0.0;  // sparse-G skip (:294-295)
                    if (!(up0 || up1)) continue;
                    const double f0 = __dmul_rn(coef, g0), f1 = __dmul_rn(coef, g1);
                    double2* row0 = reinterpret_cast<double2*>(Rb + l0 * n);
                    double2* row1 = reinterpret_cast<double2*>(Rb + (has1 ? l1 : l0) * n);
                    double acc0 = 0.0, acc1 = 0.0;
                    for (long long k0 = lane; k0 < h; k0 += 32 * kR) {
                        double2 zv[kR], r0[kR], r1[kR];
#pragma unroll
                        for (int u = 0; u < kR; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < h) {
                                zv[u] = __ldcg(z2 + k);
                                if (up0) r0[u] = __ldcg(row0 + k);
                                if (up1) r1[u] = __ldcg(row1 + k);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kR; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < h) {
                                if (up0) {
                                    double2 r;
                                    r.x = __dsub_rn(r0[u].x, __dmul_rn(f0, zv[u].x));
                                    r.y = __dsub_rn(r0[u].y, __dmul_rn(f0, zv[u].y));
                                    row0[k] = r;
                                    acc0 += r.x * r.x;
                                    acc0 += r.y * r.y;
                                }
                                if (up1) {
                                    double2 r;
                                    r.x = __dsub_rn(r1[u].x, __dmul_rn(f1, zv[u].x));
                                    r.y = __dsub_rn(r1[u].y, __dmul_rn(f1, zv[u].y));
                                    row1[k] = r;
                                    acc1 += r.x * r.x;
                                    acc1 += r.y * r.y;
                                }
                            }
                        }
                    }
                    if (up0) {
                        const double rs0 = warp_sum(acc0);
                        if (lane == 0) rsq[l0] = rs0;
                    }
                    if (up1) {
                        const double rs1 = warp_sum(acc1);
                        if (lane == 0) rsq[l1] = rs1;
                    }
                }
            } else {
                for (long long l = gw; l < m; l += nw) {
                    const double gl = coef_of(l);
                    if (gl == 0.0) continue;  // R_l unchanged (solver.hpp:294-295)
                    const double f = __dmul_rn(coef, gl);
                    double* row = Rb + l * n;
                    double acc = 0.0;
                    for (long long k0 = lane; k0 < n; k0 += 32 * kU) {
                        double rv[kU], zv[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < n) {
                                rv[u] = __ldcg(row + k);
                                zv[u] = __ldcg(zo + k);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const long long k = k0 + 32 * u;
                            if (k < n) {
                                const double r = __dsub_rn(rv[u], __dmul_rn(f, zv[u]));
                                row[k] = r;
                                acc += r * r;
                            }
                        }
                    }
                    const double rs = warp_sum(acc);
                    if (lane == 0) rsq[l] = rs;
                }
            }
            x_update(Ai, coef, sel);
        }
        PT_MARK(4);
        grid.sync();
        PT_MARK(6);
        // ---- phase D (every CTA): refresh r_sq, fixed-order reductions, finalize ----
        {
            double ps = 0.0, pm = -INFINITY, pe = 0.0;
            long long pa = LLONG_MAX;
            // loads batched 8 per thread ahead of the arithmetic: one L2 round
            // trip per 8·kT rows instead of one per kT
            for (long long i0 = tid; i0 < m; i0 += 8 * kT) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const long long i = i0 + (long long)u * kT;
                    v[u] = i < m ? __ldcg(rsq + i) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const long long i = i0 + (long long)u * kT;
                    if (i < m) {
                        rs_s[i] = v[u];
                        ps += v[u];
                        const double as = as_s[i];
                        if (as > 0.0) maxidx_merge(pm, pa, __ddiv_rn(v[u], as), i);
                    }
                }
            }
            const long long nx = x_slots;
            for (long long b0 = tid; b0 < nx; b0 += 4 * kT) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const long long b = b0 + (long long)u * kT;
                    v[u] = b < nx ? __ldcg(xpart + b) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) pe += v[u];
            }
            // one fused pass: warp trees, then thread 0 over the warps in order
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ps += __shfl_xor_sync(0xffffffffu, ps, o);
                pe += __shfl_xor_sync(0xffffffffu, pe, o);
                const double ov = __shfl_xor_sync(0xffffffffu, pm, o);
                const long long oi = __shfl_xor_sync(0xffffffffu, pa, o);
                maxidx_merge(pm, pa, ov, oi);
            }
            if (lane == 0) {
                red[warp] = ps;
                sh.scan[warp] = pe;
                sh.redv[warp] = pm;
                sh.redi[warp] = pa;
            }
            __syncthreads();
            if (tid == 0) {
                ps = 0.0;
                pe = 0.0;
                pm = -INFINITY;
                pa = LLONG_MAX;
                for (int w = 0; w < kW; ++w) {
                    ps += red[w];
                    pe += sh.scan[w];
                    maxidx_merge(pm, pa, sh.redv[w], sh.redi[w]);
                }
                if (P.a_rp) {  // CSR A: the incremental tracker, clamped (solver.hpp:290)
                    pe = __dadd_rn(lst.err_sq, pe);
                    if (pe < 0.0) pe = 0.0;
                }
                lst.r_fro_sq = ps;
                lst.max_ratio = pm;
                lst.argmax = pa;
                lst.err_sq = pe;
                lst.sel_valid = 0;
                const double cf = P.c_fro > 0.0 ? P.c_fro : 1.0;
                const double rel = sqrt(ps > 0.0 ? ps : 0.0) / cf;
                if (!isfinite(ps)) {  // solver.hpp:306-307
                    lst.status = ST_ERROR;
                    lst.err_code = 4;
                    lst.err_k = lst.k;
                    lst.err_val = sqrt(fabs(ps));
                } else if (lst.fin_mode == FIN_UPDATE_ROW) {  // no k++, trace or stop check
                    lst.metric = P.stop_kind == 0 ? pe / P.ref_sq : rel;
                    lst.k_limit = lst.k;
                } else {
                    const unsigned long long k = lst.k;
                    const double metric = P.stop_kind == 0 ? pe / P.ref_sq : rel;
                    const unsigned long long slot = k - lst.k0;
                    if (rank == 0 && slot < P.trace_cap) {
                        P.trace_row[slot] = sel;
                        P.trace_metric[slot] = metric;
                        P.trace_rel[slot] = rel;
                    }
                    lst.k = k + 1;
                    lst.metric = metric;
                    if (lst.run_mode && metric <= P.tol) lst.status = ST_PAUSE;
                    else if (lst.run_mode && !(ps > 0.0)) lst.status = ST_ZERO;
                }
            }
            __syncthreads();
        }
        PT_MARK(5);
    }
    if (P.g_rp && rank == 0 && g_prev >= 0) {  // leave g all-zero for the next launch
        __syncthreads();
        for (long long e = P.g_rp[g_prev] + tid; e < P.g_rp[g_prev + 1]; e += kT) go[P.g_ci[e]] = 0.0;
    }
    if (rank == 0 && tid == 0) *P.st = lst;
    PT_STORE();
}

template <int kT>
__global__ void __launch_bounds__(kT, 1) k_persist_lat(Params P) {
    persist_body_lat<GridGroup, kT>(P, GridGroup{cooperative_groups::this_grid()});
}

int persist_grid(const Params& P) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sizeof(double) * (size_t)((P.m + 31) / 32);
    cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_persist, kPersistThreads, smem);
    return std::max(1, sms * std::min(per, 1));
}

// K3 standalone: (re)select with the configured rule (consume=0: speculative,
// snapshot kept) or run a public select_*(θ) that consumes the stream (consume=1).
__global__ void __launch_bounds__(kThreads) k_select(Params P, int method, double theta,
                                                    int consume, long long scratch_cap) {
    extern __shared__ double scratch[];
    __shared__ SelShared sh;
    DevState* st = P.st;
    if (!consume) {
        finish_select(P, st, sh, scratch, scratch_cap);
        return;
    }
    long long row = 0;
    if (threadIdx.x == 0) sh.err = 0;
    __syncthreads();
    const int err = select_rows(P, st, method, theta, &row, sh, scratch, scratch_cap);
    __syncthreads();
    if (threadIdx.x == 0) {
        st->sel_valid = 0;
        st->q_row = row;
        if (err) {
            st->status = ST_ERROR;
            st->err_code = err;
        }
    }
}

// greedy_threshold / greedy_index_set / max_residual_ratio queries (no RNG use)
__global__ void __launch_bounds__(kThreads) k_query(Params P, double theta, int want_set) {
    __shared__ double red[kWarps];
    DevState* st = P.st;
    const double r_fro = st->r_fro_sq;
    const long long argmax = st->argmax;
    const bool zero = !(r_fro > 0.0);
    const double zeta = zero ? 0.0
                             : __dadd_rn(__dmul_rn(theta, __ddiv_rn(st->max_ratio, r_fro)),
                                         __ddiv_rn(__dsub_rn(1.0, theta), P.a_fro_sq));
    long long cnt = 0;
    if (want_set && !zero) {
        for (long long i = threadIdx.x; i < P.m; i += kThreads) {
            const double as = P.a_sq[i];
            const int mem = as > 0.0 &&
                            (i == argmax || P.r_sq[i] >= __dmul_rn(__dmul_rn(zeta, as), r_fro));
            P.member_flags[i] = mem;
            cnt += mem;
        }
    }
    const double c = block_sum((double)cnt, red);
    if (threadIdx.x == 0) {
        st->q_zeta = zeta;
        st->q_row = argmax;
        st->q_count = (long long)c;
        if (zero) {
            st->status = ST_ERROR;
            st->err_code = 2;
        }
    }
}

__global__ void k_rollback(DevState* st) {
    if (st->sel_valid) {
        for (int k = 0; k < 4; ++k) st->rng[k] = st->rng_snap[k];
        st->cyclic_pos = st->cyclic_snap;
        st->skipped_zero_rows = st->skipped_snap;
        st->sel_valid = 0;
    }
}

// fresh ‖X − X_ref‖² (solver.hpp:188, :414, :475) and the all-finite check (:428)
__global__ void __launch_bounds__(kThreads) k_err_fresh(Params P) {
    __shared__ double red[kWarps];
    __shared__ bool last;
    DevState* st = P.st;
    const long long total = P.x1r * P.q;  // this rank's rows of X: [x0r, x1r)
    double acc = 0.0, bad = 0.0;
    for (long long e = P.x0r * P.q + (long long)blockIdx.x * kThreads + threadIdx.x; e < total;
         e += (long long)gridDim.x * kThreads) {
        const double x = P.X[e];
        if (!isfinite(x)) bad += 1.0;
        if (P.Xref) {
            const double d = x - P.Xref[e];
            acc += d * d;
        }
    }
    acc = block_sum(acc, red);
    bad = block_sum(bad, red);
    if (threadIdx.x == 0) {
        P.xpart[2 * blockIdx.x] = acc;
        P.xpart[2 * blockIdx.x + 1] = bad;
        __threadfence();
        last = atomicAdd(&st->cnt_red, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0.0, b = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += kThreads) {
        s += __ldcg(P.xpart + 2 * k);
        b += __ldcg(P.xpart + 2 * k + 1);
    }
    s = block_sum(s, red);
    b = block_sum(b, red);
    if (threadIdx.x == 0) {
        st->err_sq = s;
        st->x_finite = b == 0.0;
        st->cnt_red = 0u;
        if (P.stop_kind == 0) st->metric = s / P.ref_sq;
    }
}

// ---- power iteration helpers (decomp.hpp:207-239 on the device) ----
__global__ void __launch_bounds__(kThreads) k_rowdot(const double* M, long long rows,
                                                    long long cols, const double* v, double* out) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const bool v2 = (cols & 1) == 0;
    for (long long r = warp; r < rows; r += nw) {
        const double a = warp_dot(M + r * cols, v, cols, lane, v2);
        if (lane == 0) out[r] = a;
    }
}

__global__ void __launch_bounds__(kThreads) k_coldot(const double* M, long long rows,
                                                    long long cols, const double* v, double* out,
                                                    double* part, unsigned int* cnt, int nslab,
                                                    int nj, int jrows) {
    __shared__ bool last;
    const int slab = blockIdx.x % nslab, jc = blockIdx.x / nslab;
    const long long j0 = (long long)jc * jrows, j1 = min(rows, j0 + jrows);
    const long long c = (long long)slab * kThreads + threadIdx.x;
    double a = 0.0;
    if (c < cols)
        for (long long j = j0; j < j1; ++j) a += __ldg(v + j) * __ldg(M + j * cols + c);
    if (nj == 1) {
        if (c < cols) out[c] = a;
        return;
    }
    if (c < cols) part[(long long)jc * cols + c] = a;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(cnt + slab, 1u) == (unsigned)(nj - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (c < cols) {
        double s = 0.0;
        for (int k = 0; k < nj; ++k) s += __ldcg(part + (long long)k * cols + c);
        out[c] = s;
    }
    if (threadIdx.x == 0) cnt[slab] = 0u;
}

// rayleigh = v·w, wn = ‖w‖, v_out = w / wn   (decomp.hpp:227-231)
__global__ void __launch_bounds__(1024) k_power_step(const double* v, const double* w,
                                                     double* v_out, long long dim, double* out2) {
    __shared__ double red[32];
    __shared__ double wn_s;
    double a = 0.0, b = 0.0;
    for (long long i = threadIdx.x; i < dim; i += blockDim.x) {
        a += v[i] * w[i];
        b += w[i] * w[i];
    }
    a = block_sum(a, red);
    b = block_sum(b, red);
    if (threadIdx.x == 0) {
        wn_s = sqrt(b);
        out2[0] = a;
        out2[1] = wn_s;
    }
    __syncthreads();
    const double wn = wn_s;
    if (wn != 0.0)
        for (long long i = threadIdx.x; i < dim; i += blockDim.x) v_out[i] = w[i] / wn;
}

// Power-iteration step on a small Gram M (w = M·v already formed), with the
// reference's stop test on the device (decomp.hpp:227-238):
//   rayleigh = v·w, wn = ‖w‖, v ← w / wn; stop when it > 0 and
//   |rayleigh − λ| ≤ ½·tol·|rayleigh|  →  ‖B‖₂ = √rayleigh.
// ps: [0] λ, [1] result, [2] iteration, [3] state (0 running, 1 done, 2 cap hit)
__global__ void __launch_bounds__(1024) k_power_step2(double* v, const double* w, long long dim,
                                                      double* ps, double tol, double max_iter) {
    __shared__ double red[32];
    __shared__ int stop;
    if (ps[3] != 0.0) return;
    double a = 0.0, b = 0.0;
    for (long long i = threadIdx.x; i < dim; i += blockDim.x) {
        a += v[i] * w[i];
        b += w[i] * w[i];
    }
    a = block_sum(a, red);
    b = block_sum(b, red);
    const double wn = sqrt(b);
    if (threadIdx.x == 0) {
        stop = 0;
        if (wn == 0.0) {
            ps[1] = 0.0;
            ps[3] = 1.0;
            stop = 1;
        } else {
            const double it = ps[2];
            if (it > 0.0 && fabs(a - ps[0]) <= 0.5 * tol * fabs(a)) {
                ps[1] = sqrt(a);
                ps[3] = 1.0;
            } else {
                ps[0] = a;
                if (it + 1.0 >= max_iter) ps[3] = 2.0;
            }
            ps[2] = it + 1.0;
        }
    }
    __syncthreads();
    if (stop) return;
    for (long long i = threadIdx.x; i < dim; i += blockDim.x) v[i] = w[i] / wn;
}

// out (cols × rows) = inᵀ, 32×32 smem tiles
__global__ void k_transpose(const double* in, long long rows, long long cols, double* out) {
    __shared__ double t[32][33];
    const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const long long r = r0 + j, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[j][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const long long c = c0 + j, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = t[threadIdx.x][j];
    }
}

__global__ void k_fill(double* p, long long n, double v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

// host → device control writes for a batch (one launch instead of several memcpys)
__global__ void k_ctrl(DevState* st, unsigned long long k0, unsigned long long k_limit,
                       int fin_mode, int run_mode, int reset_status) {
    st->k0 = k0;
    st->k_limit = k_limit;
    st->fin_mode = fin_mode;
    st->run_mode = run_mode;
    if (reset_status) {
        st->status = ST_RUN;
        st->err_code = 0;
    }
}

__global__ void k_set_replay(DevState* st, int on) { st->replay = on; }

__global__ void k_set_sel(DevState* st, long long sel, double coef) {
    st->sel = sel;
    st->coef = coef;
    st->sel_valid = 0;
}

// per-CTA Σ v² partials (deterministic), reduced by k_reduce_parts (axb_gemm.cu)
__global__ void __launch_bounds__(kThreads) k_sumsq(const double* v, long long n, double* part) {
    __shared__ double red[kWarps];
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kThreads) {
        const double x = v[i];
        acc += x * x;
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// ‖A_i‖² per row with the reference's sequential order and rounding
// (matrix.hpp:300-306 via RowView::sq_norm :199-203): one thread per row.
__global__ void k_row_sq_seq(const double* A, long long m, long long p, double* out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
        const double* row = A + i * p;
        double s = 0.0;
        for (long long j = 0; j < p; ++j) {
            const double v = row[j];
            s = __dadd_rn(s, __dmul_rn(v, v));
        }
        out[i] = s;
    }
}

// a_fro_sq and the RBK inclusive cumsum, sequential as solver.hpp:157-166
__global__ void k_cumsum_seq(const double* a_sq, long long m, double* cum, double* total) {
    double c = 0.0;
    for (long long i = 0; i < m; ++i) {
        c = __dadd_rn(c, a_sq[i]);
        cum[i] = c;
    }
    *total = c;
}

}  // namespace

// copy out (and optionally reset) the timeline ring; zeros unless built with
// -DAXB_TRACE_TIMELINE
int timeline_read(unsigned long long* out, int reset) {
#ifdef AXB_TRACE_TIMELINE
    if (out && cudaMemcpyFromSymbol(out, g_axb_tl, sizeof(unsigned long long) * 64 * 8) != cudaSuccess)
        return 0;
    if (reset) {
        static unsigned long long init[64][8];
        for (int i = 0; i < 64; ++i)
            for (int j = 0; j < 8; ++j) init[i][j] = (j & 1) ? 0ull : ~0ull;
        cudaMemcpyToSymbol(g_axb_tl, init, sizeof init);
    }
    return 1;
#else
    if (out)
        for (int i = 0; i < 64 * 8; ++i) out[i] = 0ull;
    (void)reset;
    return 0;
#endif
}


// ------------------------------------------------------------------------
// launchers

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

void launch_yg(const Params& P, cudaStream_t s, bool with_g) {
    if (P.yg_tma) {
        const size_t smem = (size_t)P.r_stages * P.r_chunk * 16 + 2 * P.r_stages * 8;
        static size_t attr_set[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (attr_set[dev & 63] < smem) {
            cudaFuncSetAttribute(k_yg_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr_set[dev & 63] = smem;
        }
        launch_pdl(k_yg_tma, P.r_grid, kTmaThreads, smem, s, P, with_g ? 1 : 0);
        return;
    }
    launch_pdl(k_yg, P.yg_grid, kYgThreads, 0, s, P, with_g ? 1 : 0);
}

void launch_zx(const Params& P, cudaStream_t s) {
    launch_pdl(k_zx, P.z_nslab * P.z_nj + P.x_ctas, kThreads, 0, s, P);
}

void launch_r(const Params& P, cudaStream_t s, bool update) {
    if (P.r_tma) {
        const size_t smem = tma_smem_bytes(P);
        static size_t attr_set[64] = {};  // function attributes are per device
        int dev = 0;
        cudaGetDevice(&dev);
        size_t& done = attr_set[dev & 63];
        if (done < smem) {  // opt in up to (device limit − static smem)
            int optin = 0;
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, k_r_tma<true>);
            const int dyn = optin - (int)fa.sharedSizeBytes;
            cudaFuncSetAttribute(k_r_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            cudaFuncSetAttribute(k_r_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            // one shared-memory carve-out for all three iteration kernels, so
            // consecutive (PDL-overlapped) launches never reconfigure L1/smem
            // — sized for K2's CTAs only: a larger carve-out (room for the k_zx
            // CTAs' y staging too) measured slower, k_zx wants the L1
            const int cps = std::max(1, (P.r_grid + 147) / 148);
            int pct = (int)((100.0 * cps * (smem + fa.sharedSizeBytes + 1024)) / optin + 0.999);
            pct = std::min(100, std::max(pct, 1));
            if (const char* e = std::getenv("AXB_CARVEOUT")) pct = std::atoi(e);
            cudaFuncSetAttribute(k_r_tma<true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            cudaFuncSetAttribute(k_r_tma<false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            cudaFuncSetAttribute(k_yg, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            cudaFuncSetAttribute(k_yg_tma, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            cudaFuncSetAttribute(k_zx, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            done = (size_t)dyn;
        }
        if (update) launch_pdl(k_r_tma<true>, P.r_grid, kTmaThreads, smem, s, P);
        else k_r_tma<false><<<P.r_grid, kTmaThreads, smem, s>>>(P);
        return;
    }
    const size_t smem = sizeof(double) * (size_t)(P.r_chunk + P.r_rows_per_cta);
    const bool v2 = (P.n & 1) == 0;
    if (update) {
        if (v2) k_r<true, true><<<P.r_grid, kThreads, smem, s>>>(P);
        else k_r<true, false><<<P.r_grid, kThreads, smem, s>>>(P);
    } else {
        if (v2) k_r<false, true><<<P.r_grid, kThreads, smem, s>>>(P);
        else k_r<false, false><<<P.r_grid, kThreads, smem, s>>>(P);
    }
}

void launch_select(const Params& P, cudaStream_t s, int method, double theta, int consume) {
    const long long ng = (P.m + 31) / 32;
    const long long cap = ng <= 4096 ? ng : 0;  // group sums in ≤32 KB of smem, else P.gsum
    k_select<<<1, kThreads, (size_t)cap * 8, s>>>(P, method, theta, consume, cap);
}

void launch_query(const Params& P, cudaStream_t s, double theta, int want_set) {
    k_query<<<1, kThreads, 0, s>>>(P, theta, want_set);
}

void launch_rollback(const Params& P, cudaStream_t s) { k_rollback<<<1, 1, 0, s>>>(P.st); }

void launch_err_fresh(const Params& P, cudaStream_t s) {
    long long total = P.p * P.q;
    int grid = (int)std::min<long long>(296, (total + kThreads * 4 - 1) / (kThreads * 4));
    if (grid < 1) grid = 1;
    k_err_fresh<<<grid, kThreads, 0, s>>>(P);
}

void launch_rowdot(const double* M, long long rows, long long cols, const double* v, double* out,
                   cudaStream_t s) {
    int grid = (int)std::min<long long>(148 * 8, (rows + kWarps - 1) / kWarps);
    k_rowdot<<<grid, kThreads, 0, s>>>(M, rows, cols, v, out);
}

void launch_coldot(const double* M, long long rows, long long cols, const double* v, double* out,
                   double* part, unsigned int* cnt, int nj, int jrows, cudaStream_t s) {
    const int nslab = (int)((cols + kThreads - 1) / kThreads);
    k_coldot<<<nslab * nj, kThreads, 0, s>>>(M, rows, cols, v, out, part, cnt, nslab, nj, jrows);
}

void launch_power_step(const double* v_in, const double* w, double* v_out, long long dim,
                       double* out2, cudaStream_t s) {
    k_power_step<<<1, 1024, 0, s>>>(v_in, w, v_out, dim, out2);
}

void launch_ctrl(DevState* st, unsigned long long k0, unsigned long long k_limit, int fin_mode,
                 int run_mode, int reset_status, cudaStream_t s) {
    k_ctrl<<<1, 1, 0, s>>>(st, k0, k_limit, fin_mode, run_mode, reset_status);
}

void launch_set_replay(DevState* st, int on, cudaStream_t s) { k_set_replay<<<1, 1, 0, s>>>(st, on); }

void launch_set_sel(DevState* st, long long sel, double coef, cudaStream_t s) {
    k_set_sel<<<1, 1, 0, s>>>(st, sel, coef);
}

int sumsq_parts(long long n) { return (int)std::max<long long>(1, std::min<long long>(1184, (n + 1023) / 1024)); }

void launch_sumsq(const double* v, long long n, double* part, cudaStream_t s) {
    k_sumsq<<<sumsq_parts(n), kThreads, 0, s>>>(v, n, part);
}

void launch_row_sq_seq(const double* A, long long m, long long p, double* out, cudaStream_t s) {
    int grid = (int)std::max<long long>(1, std::min<long long>(148 * 8, (m + 127) / 128));
    k_row_sq_seq<<<grid, 128, 0, s>>>(A, m, p, out);
}

void launch_cumsum_seq(const double* a_sq, long long m, double* cum, double* total, cudaStream_t s) {
    k_cumsum_seq<<<1, 1, 0, s>>>(a_sq, m, cum, total);
}

// k_sel1 (global reductions, stop logic, selection) then, when it selects,
// k_pack (the owner's row copy)
void launch_sel1(const Params& P, cudaStream_t s, int mode) {
    k_sel1<<<std::max(1, P.sel1_grid), kThreads, 0, s>>>(P, mode);
    if (mode != 0) launch_pdl(k_pack, std::max(1, P.pack_grid), kThreads, 0, s, P);
}

void launch_power_step2(double* v, const double* w, long long dim, double* ps, double tol,
                        double max_iter, cudaStream_t s) {
    k_power_step2<<<1, 1024, 0, s>>>(v, w, dim, ps, tol, max_iter);
}

void launch_transpose(const double* in, long long rows, long long cols, double* out,
                      cudaStream_t s) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out);
}

void launch_sel_greedy(const Params& P, cudaStream_t s) {
    launch_pdl(k_sel_greedy, P.sel_grid, kThreads, 0, s, P);
}

// (batched systems run the general body: one CTA owns a system, so the latency
// body's per-CTA refresh of every r_sq buys nothing there — measured slower)
int launch_persist_batch(const Params* dPs, int count, long long max_m, cudaStream_t s) {
    const size_t smem = sizeof(double) * (size_t)((max_m + 31) / 32);
    // static shared memory counts against the 48 KB default too: always opt in
    // two 256-thread systems per SM once there are at least two per SM: one CTA's
    // serial phases (selection, reductions) then overlap the other's streaming.
    // Config-1 systems, 2000 steps (tools/prof_batch.py): 296 / 592 systems
    // 845k → 869k / 847k → 874k it/s; 148 systems stay on 512 threads (615k on 256)
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* e = getenv("AXB_BATCH_THREADS");
    const int forced = e ? atoi(e) : 0;
    const int threads = (forced == 256 || forced == 512 || forced == 1024) ? forced
                        : (count >= 2 * sms ? 256 : kBatchThreads);
    if (threads == 256) {
        cudaFuncSetAttribute(k_persist_batch<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_persist_batch<256><<<count, 256, smem, s>>>(dPs);
    } else if (threads == 1024) {
        cudaFuncSetAttribute(k_persist_batch<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_persist_batch<1024><<<count, 1024, smem, s>>>(dPs);
    } else {
        cudaFuncSetAttribute(k_persist_batch<kBatchThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        k_persist_batch<kBatchThreads><<<count, kBatchThreads, smem, s>>>(dPs);
    }
    return (int)cudaGetLastError();
}

int launch_persist(const Params& P, cudaStream_t s) {
    if (P.persist_lat) {
        const int threads = P.persist_lat == 128 ? 128 : 256;
        const void* fn = threads == 128 ? (const void*)k_persist_lat<128> : (const void*)k_persist_lat<256>;
        const size_t smem = sizeof(double) * persist_lat_smem_doubles(P.m, threads);
        // always opt in: the kernel's static shared memory (state copy, scan
        // scratch) counts against the same 48 KB default — m = 2000 (48.5 KB
        // dynamic + ~3 KB static) failed the cooperative launch without it
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
        const int grid = std::min(P.persist_grid, std::max(1, sms * std::min(per, 1)));
        Params Pc = P;
        void* args[] = {&Pc};
        return (int)cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(threads), args,
                                                smem, s);
    }
    const int grid = std::min(P.persist_grid, persist_grid(P));
    const size_t smem = sizeof(double) * (size_t)((P.m + 31) / 32);
    cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    Params Pc = P;
    void* args[] = {&Pc};
    return (int)cudaLaunchCooperativeKernel((const void*)k_persist, dim3((unsigned)grid),
                                            dim3(kPersistThreads), args, smem, s);
}

__global__ void __launch_bounds__(256) k_spmm_csr(const long long* __restrict__ rp,
                                                  const int* __restrict__ ci,
                                                  const double* __restrict__ v, long long rows,
                                                  const double* __restrict__ X, long long q,
                                                  double* __restrict__ T) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = w; i < rows; i += nw) {
        const long long e0 = rp[i], e1 = rp[i + 1];
        for (long long c = lane; c < q; c += 32) {
            double a = 0.0;
            for (long long e = e0; e < e1; ++e) a = __dadd_rn(a, __dmul_rn(v[e], X[(long long)ci[e] * q + c]));
            T[i * q + c] = a;
        }
    }
}

void launch_spmm_csr(const long long* rp, const int* ci, const double* v, long long rows,
                     const double* X, long long q, double* T, cudaStream_t s) {
    const int grid = (int)std::max<long long>(1, std::min<long long>(148 * 8, (rows + 7) / 8));
    k_spmm_csr<<<grid, 256, 0, s>>>(rp, ci, v, rows, X, q, T);
}

void launch_fill(double* p, long long n, double v, cudaStream_t s) {
    int grid = (int)std::min<long long>(1184, (n + 255) / 256);
    if (grid < 1) grid = 1;
    k_fill<<<grid, 256, 0, s>>>(p, n, v);
}

}  // namespace axb_dev

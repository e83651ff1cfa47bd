// K2-TC: back-projection on the 5th-generation tensor cores (tcgen05).
// Replaces fbp.back_project (fbp.py:186-252) on the default path.
//
// For one angle, a tile of 121 voxel columns (11 x 11, padded to the MMA's
// M = 128) and NR detector rows, back-projection is a small GEMM
//     D[m][z] += sum_k W[m][k] * T[k][z],
// T the feathered filtered taps of the tile's channel window [c_lo, c_lo+16)
// and W the interpolation matrix: row m holds voxel m's exact two-tap weights
// {1 - f, f} at k = floor(t) - c_lo and k + 1, zeros elsewhere
// (fbp.py:237-245).  Summed over the angles, D is the unscaled
// back-projection.  The tile's window spans 10 (|cos| + |sin|) + 1 <= 15.2
// channels, so 97% of the angles need one K = 16 "item"; the others need two
// (channels c_lo + [0, 16) and [16, 32)).
//
// Precision: fp32 operands are split into fp16 pairs (hi + lo, 22
// significant bits); D accumulates W_hi T_hi + W_lo T_hi + W_hi T_lo in fp32
// TMEM (the dropped W_lo T_lo is < 2^-22 relative).  The taps of detector
// row z are scaled by 2^e[z] so they sit in fp16's normal range; the
// epilogue multiplies by 2^-e[z] exactly.  e[z] is per ROW, so a row's result
// depends on that row's data only (row independence, test_fbp.py:180-191).
// The tensor core's fp32 accumulation truncates, so D holds blocks of 16
// angles -- blocks of the ABSOLUTE angle index (k / 16), so chained angle
// chunks at multiples of 16 sum exactly like one pass -- and each finished
// block is added with round-to-nearest into a master sum kept in the weight
// warps' registers.
//
// CTA (576 threads, one per SM, persistent) = one 11 x 11 tile x NR rows per
// round (NR = 256, or 128 for short slabs), TMEM = two ping-pong accumulators
// of NR columns:
//   warp 0      prefetches the tensor map;
//   warp 1      TMEM owner and MMA issuer: per item, one elected lane issues 3
//               tcgen05.mma.kind::f16 (A = W from shared memory, K-major; B =
//               T, MN-major), one tcgen05.commit frees the slot; the item's
//               flags arrive in a control word with the slot;
//   warps 2-17  four weight groups of 4 warps (group g: angles = g mod 4; one
//               voxel row per thread): fp32 t relative to the fp64 window
//               origin, the fp16 hi/lo W rows stored to the slot's A tiles;
//               the group's lane-quadrant-0 warp also issues the item's tap
//               box (one cp.async.bulk.tensor: T_hi and T_lo, 16 channels x
//               NR rows, MN-major canonical layout; the OOB zero fill is the
//               reference's zero guard for off-detector taps) and writes its
//               control word.  Every warp also owns NR/4 columns of the RN
//               master sum of its 32 voxels (64 registers at NR = 256): it
//               flushes finished blocks (tcgen05.ld + fadd.rn) and writes the
//               epilogue (x 2^-e, FoV mask and angle weight, fbp.py:247-251).
// The tap ring and the weight ring share one "full" mbarrier per slot (TMA
// transaction bytes + 4 weight-warp arrivals) and one "empty" barrier (the
// MMA commit), so the MMA warp waits once per item.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cuda_fp16.h>

#include "bp_plan.hpp"
#include "common.cuh"

namespace tf {
namespace {

constexpr int kTX = kTileShape[kShapeTc][0], kTY = kTileShape[kShapeTc][1], kMV = kTX * kTY;
constexpr int kM = 128;         // MMA M = TMEM lanes: voxel rows of the tile
constexpr int kK = 16;          // channels per item (one fp16 MMA K-step)
#ifndef TF_TC_S
#define TF_TC_S 8
#endif
constexpr int kS = TF_TC_S;     // ring depth in items
#ifndef TF_TC_P
#define TF_TC_P 16
#endif
constexpr int kP = TF_TC_P;     // angles per accumulator block (absolute angle index / kP)
constexpr int kG = 4;           // weight groups of 4 warps
constexpr int kThreads = 64 + 128 * kG;
#ifndef TF_TC_LAG
#define TF_TC_LAG 14
#endif
// a group flushes block j before it produces its first angle >= end(j) + kLag: by then the group's own
// slot waits proved block j's MMAs retired (no wait on accfull), and every group still flushes before
// the MMA warp needs the accumulator again at angle end(j) + kP (kLag <= kP: no group has to wait for
// a slot the MMA warp could only free after that)
constexpr int kLag = TF_TC_LAG;
static_assert(kLag <= kP, "a block is flushed before its accumulator is needed again");
constexpr int kWPlane = kM * kK * 2;   // one fp16 plane of a slot's W tile (4 KB)
constexpr float kOneStep = 14.9f;      // window test (fp32 margin below 15)
static_assert(kMV <= kM, "tile fits the MMA's M");
static_assert(32 % kG == 0, "a batch of 32 angles splits evenly over the groups");

template <int NR>
struct TcCfg {
    static constexpr int TAP_PLANE = NR * kK * 2;                   // one fp16 plane of a slot's taps
    static constexpr int SLOT = 2 * TAP_PLANE + 2 * kWPlane;        // taps hi, lo + W hi, lo
    static constexpr int NC = NR / kG;                              // master columns per thread
    static constexpr int SMEM = kS * SLOT + NR * 8 + (2 * kS + 4) * 8 + 16 + 4 * kS;
    static constexpr uint32_t TMEM_COLS = 2 * NR;
};

struct TCArgs {
    const double2* trig;
    const int* tiles;   // work list: FoV-active tiles (Morton order) of one z-block
    int n_tiles, n_work;  // tiles per z-block; work items = z-blocks x n_tiles
    unsigned* sync;     // grid-barrier counter of the lockstep rounds (workspace header, zeroed per call)
    const int* e_rows;  // per-row tap exponent (workspace header)
    float* vol;
    int a0, a1, ws_a0, n_rows, nx, ny;
    int x0, x1, y0, y1;
    int ntx, flags;
    double cx, cy, scale, axis, R2, sc2;
    float angle_wf;
#ifdef TF_TC_PROBE
    long long* probe;  // tools/tc_probe.cu: per-CTA wait-cycle counters (never in the product library)
#endif
};

#ifdef TF_TC_PROBE
#define PROBE_T0(v) const long long v = clock64()
#define PROBE_ADD(acc, t0) acc += clock64() - (t0)
#else
#define PROBE_T0(v)
#define PROBE_ADD(acc, t0)
#endif

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100); SWIZZLE_NONE, base offset 0
    return d;
}

__device__ __forceinline__ void umma_f16_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
    return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

#define TC_LD16(ta, v)                                                                                            \
    asm volatile(                                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),          \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])     \
        : "r"(ta))

// the tile's channel window for one angle: the fp64 tile-origin coordinate
// (geometry.py:148-153 operation order) and c_lo = floor of its minimum over
// the tile; threads add fp32 offsets to F0 = t0 - c_lo
struct TcWin {
    int c_lo;
    float F0, B, C;
};
__device__ __forceinline__ TcWin tc_window(double dX, double dY, double2 cs, const TCArgs& a) {
    double t0 = __dadd_rn(__dmul_rn(dX, cs.x), __dmul_rn(dY, cs.y));
    t0 = __dadd_rn(__dmul_rn(t0, a.scale), a.axis);
    const double B = cs.x * a.scale, C = cs.y * a.scale;
    const double tmin = t0 + fmin(0.0, B * (kTX - 1)) + fmin(0.0, C * (kTY - 1));
    TcWin w;
    w.c_lo = (int)floor(tmin);
    w.F0 = (float)(t0 - (double)w.c_lo);
    w.B = (float)B;
    w.C = (float)C;
    return w;
}
// one item when every tap of the tile lies in the window's first 16 channels
__device__ __forceinline__ bool tc_two_items(const TcWin& w) {
    const float span = w.F0 + fmaxf(0.f, w.B * (kTX - 1)) + fmaxf(0.f, w.C * (kTY - 1));
    return !(span < kOneStep);
}
__device__ __forceinline__ TcWin tc_bcast(const TcWin& w, int src) {
    TcWin r;
    r.c_lo = __shfl_sync(0xffffffffu, w.c_lo, src);
    r.F0 = __shfl_sync(0xffffffffu, w.F0, src);
    r.B = __shfl_sync(0xffffffffu, w.B, src);
    r.C = __shfl_sync(0xffffffffu, w.C, src);
    return r;
}

// 32 consecutive angles g0 + lane: each lane's window and the warp-wide mask
// of the angles that need two items (every role walks the same item sequence)
struct TcBatch {
    TcWin w;
    uint32_t two;
    int n;  // angles in the batch
};
__device__ __forceinline__ TcBatch tc_batch(int g0, int n_ang, double dX, double dY, const TCArgs& a) {
    const int lane = threadIdx.x & 31;
    const int g = min(g0 + lane, n_ang - 1);
    TcBatch b;
    b.w = tc_window(dX, dY, a.trig[a.a0 + g], a);
    b.two = __ballot_sync(0xffffffffu, g0 + lane < n_ang && tc_two_items(b.w));
    b.n = min(32, n_ang - g0);
    return b;
}

__device__ __forceinline__ bool tc_outside_fov(int x, int y, const TCArgs& a) {
    // ((x-cx)^2 + (y-cy)^2) * scale^2 > R^2, no FMA contraction (fbp.py:247-250)
    double dx = __dsub_rn((double)x, a.cx), dy = __dsub_rn((double)y, a.cy);
    double rr = __dmul_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), a.sc2);
    return rr > a.R2;
}

// Persistent, lockstep: the grid is one CTA per SM (cooperative launch) and
// CTA b processes the work items w = r G + b (r = 0, 1, ...) of the list of
// (z-block, FoV-active tile) pairs, z-block outer, tiles in Morton order.  A
// grid-wide barrier between rounds keeps the G CTAs of a round -- a compact
// patch of Morton-adjacent tiles -- at the same angle within a few percent,
// so the patch's tap windows are fetched from DRAM once and re-read from L2
// by its other CTAs (a grid of one CTA per tile let resident CTAs sit at
// unrelated angles: 2.4 TB of DRAM reads per C3 volume, 62% L2 hits).  The
// ring slots, their phases and the accumulator ping-pong run on across the
// rounds; each round resets the RN master sum and ends with the epilogue.
template <int NR>
__global__ void __launch_bounds__(kThreads, 1) bp_tc_kernel(const __grid_constant__ CUtensorMap map, const TCArgs a) {
    using Cfg = TcCfg<NR>;
    constexpr int NC = Cfg::NC;
    extern __shared__ __align__(1024) uint8_t smem[];
    const size_t plane = (size_t)a.nx * a.ny;
    const int G = gridDim.x;
    const int n_rounds = a.n_work > (int)blockIdx.x ? (a.n_work - 1 - (int)blockIdx.x) / G + 1 : 0;

    uint8_t* const ring = smem;  // [kS] slots: T_hi, T_lo, W_hi, W_lo
    float* s_up = reinterpret_cast<float*>(ring + kS * Cfg::SLOT);  // per row of the round: 2^e and 2^-e
    float* s_dn = s_up + NR;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_dn + NR);
    uint64_t* empty = full + kS;
    uint64_t* accfull = empty + kS;   // [2]: block's MMAs done -> flush
    uint64_t* accfree = accfull + 2;  // [2]: block flushed by all 16 weight warps -> accumulator reusable
    uint32_t* tslot = reinterpret_cast<uint32_t*>(accfree + 2);
    uint32_t* s_ctl = tslot + 4;  // [kS]: the slot's item control word (written by its producer group)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
#ifdef TF_TC_PROBE_W_NONE  // probe builds only: weight warps absent from the ring
            mbar_init(&full[s], 1);
#else
            mbar_init(&full[s], 1 + 4);  // the group's TMA arrive.expect_tx + its 4 warps
#endif
            mbar_init(&empty[s], 1);     // MMA commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accfull[b], 1);
            mbar_init(&accfree[b], 4 * kG);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "n"(Cfg::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;  // columns [0, NR) accumulator 0, [NR, 2 NR) accumulator 1
    const int n_ang = a.a1 - a.a0;
    const int blk0 = a.a0 / kP;  // first absolute block
    const int n_blk = n_ang > 0 ? (a.a1 - 1) / kP - blk0 + 1 : 0;

    if (warp == 0) {
        if (lane == 0) tma_prefetch_desc(&map);
    } else if (warp == 1) {
        // ---- MMA issue: the warp runs the loop (waits are warp-uniform), one elected lane issues
        if (n_ang > 0 && n_rounds > 0) {
            // D f32, A = W f16 K-major (smem), B = T f16 MN-major (smem), M = 128, N = NR
            constexpr uint32_t idesc =
                (1u << 4) | (1u << 16) | ((uint32_t)(NR >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
            // A (K-major, no swizzle): core matrices of 8 voxel rows x 16 B, LBO = 128 B between the
            // two 8-channel chunks, SBO = 256 B between 8-row groups.  B (MN-major, no swizzle, the TMA
            // box [row/8][chan][row%8]): LBO = 128 B between 8-channel chunks, SBO = 256 B between
            // 8-row groups.  Slot offsets are added to the 14-bit start-address field (addr >> 4).
            const uint64_t dT = umma_sdesc(smem_u32(ring), 128, 256);
            const uint64_t dW = umma_sdesc(smem_u32(ring + 2 * Cfg::TAP_PLANE), 128, 256);
            int it = 0;
            long long p_full = 0, p_free = 0, p_issue = 0;
            PROBE_T0(p_start);
            // the loop does no index arithmetic of its own: each item's flags come with it (s_ctl),
            // so the warp returns to the next full-barrier wait right after issuing
            for (;; ++it) {
                const int s = it % kS;
                PROBE_T0(q1);
#ifndef TF_TC_PROBE_MMA_NOWAIT  // probe builds only: MMAs on whatever the slot holds
                mbar_wait(&full[s], (uint32_t)(it / kS) & 1u);
#endif
                PROBE_ADD(p_full, q1);
                const uint32_t ctl = *reinterpret_cast<volatile uint32_t*>(&s_ctl[s]);
                const uint32_t acc = (ctl >> 2) & 1u;
                PROBE_T0(q0);
#ifndef TF_TC_PROBE_NO_ACCFREE  // probe builds only
                if (ctl & 16u) mbar_wait(&accfree[acc], (ctl >> 5) & 1u);
#endif
                PROBE_ADD(p_free, q0);
                PROBE_T0(q2);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t so = (uint64_t)((s * Cfg::SLOT) >> 4);
                    const uint64_t th = dT + so, tl = th + (Cfg::TAP_PLANE >> 4);
                    const uint64_t wh = dW + so, wl = wh + (kWPlane >> 4);
                    const uint32_t td = tmem + acc * NR;
#ifndef TF_TC_PROBE_NO_MMA  // probe builds only: timing without the MMAs
                    umma_f16_ss(td, wh, th, idesc, (ctl & 1u) ? 0u : 1u);
#ifndef TF_TC_PROBE_NO_WLO  // probe builds only: precision experiment without the W_lo T_hi product
                    umma_f16_ss(td, wl, th, idesc, 1u);
#endif
                    umma_f16_ss(td, wh, tl, idesc, 1u);
#else
                    (void)td, (void)wh, (void)wl, (void)th, (void)tl;
#endif
                    umma_commit(&empty[s]);  // frees the slot's taps and weights
                    if (ctl & 2u) umma_commit(&accfull[acc]);
                }
                __syncwarp();
                PROBE_ADD(p_issue, q2);
                if (ctl & 8u) break;
            }
            ++it;
#ifdef TF_TC_PROBE
            if (a.probe && lane == 0 && blockIdx.x < 1024) {
                a.probe[blockIdx.x * 16 + 2] = clock64() - p_start;
                a.probe[blockIdx.x * 16 + 3] = p_full;
                a.probe[blockIdx.x * 16 + 4] = p_free;
                a.probe[blockIdx.x * 16 + 5] = p_issue;
                a.probe[blockIdx.x * 16 + 6] = it;
            }
#endif
            (void)p_full, (void)p_free, (void)p_issue;
        }
    } else {
#ifdef TF_TC_PROBE_W_NONE
        if (true) goto probe_done;
#endif
        // ---- weight groups: angle g -> group g % kG (a batch of 32 splits evenly); one voxel row
        // per thread (TMEM lane quadrant = warp % 4); column slice grp of the master sum
        const int grp = (warp - 2) >> 2;
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const bool real = m < kMV;  // rows kMV..127 of the MMA: zero weights, no output
        const int vx = m % kTX, vy = m / kTX;
        const float fdx = (float)vx, fdy = (float)vy;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);  // this warp's TMEM lanes
        const uint32_t wslot0 = smem_u32(ring + 2 * Cfg::TAP_PLANE) + (uint32_t)((m >> 3) * 256 + (m & 7) * 16);
        int it_round = 0;   // items before this round (every group counts the same sequence)
        int blk_round = 0;  // accumulator blocks before this round (the ping-pong parity runs on)
        long long p_empty = 0, p_flush = 0, p_tail = 0;
        PROBE_T0(p_start);
        for (int r = 0; r < n_rounds; ++r) {
            const int wi = r * G + (int)blockIdx.x;
            const int zb = wi / a.n_tiles;
            const int tile = a.tiles[wi - zb * a.n_tiles];
            const int zr0 = zb * NR;
            // this thread's voxel (x, y) inside the requested tile?  Recomputed for the epilogue
            // rather than kept live through the angle loop (register pressure)
            auto voxel = [&](int& x, int& y) {
                x = (tile % a.ntx) * kTX + vx;
                y = (tile / a.ntx) * kTY + vy;
                return real && x < a.nx && y < a.ny && x >= a.x0 && x < a.x1 && y >= a.y0 && y < a.y1;
            };
            const double dX = (double)((tile % a.ntx) * kTX) - a.cx, dY = (double)((tile / a.ntx) * kTY) - a.cy;
            // this round's per-row scalings (the previous round's epilogue is done with them)
            named_bar_sync(1, 128 * kG);
            for (int i = threadIdx.x - 64; i < NR; i += 128 * kG) {
                const int e = zr0 + i < a.n_rows ? a.e_rows[zr0 + i] : 0;  // |e| <= 100: normal powers of two
                s_up[i] = __int_as_float((127 + e) << 23);
                s_dn[i] = __int_as_float((127 - e) << 23);
            }
            named_bar_sync(1, 128 * kG);
            float master[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) master[j] = 0.f;
            if (a.flags & TF_BP_ACCUMULATE) {  // continue unscaled partial sums: x 2^e is exact
                int x, y;
                if (voxel(x, y)) {
                    const int zc0 = zr0 + grp * NC;
                    const float* src = a.vol + (size_t)y * a.nx + x;
#pragma unroll
                    for (int j = 0; j < NC; ++j)
                        if (zc0 + j < a.n_rows) master[j] = src[(size_t)(zc0 + j) * plane] * s_up[grp * NC + j];
                }
            }
            auto flush = [&](int lb) {  // master (+)= accumulator of block lb of the round, round to nearest
                const int gb = blk_round + lb, acc = gb & 1;
                mbar_wait(&accfull[acc], (uint32_t)(gb >> 1) & 1u);
                tc_fence_after();
#ifndef TF_TC_PROBE_NO_FLUSH  // probe builds only: timing without the TMEM reads
#pragma unroll
                for (int c = 0; c < NC; c += 16) {
                    uint32_t v[16];
                    TC_LD16(tl + (uint32_t)(acc * NR + grp * NC + c), v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 16; ++j) master[c + j] = __fadd_rn(master[c + j], __uint_as_float(v[j]));
                }
#endif
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&accfree[acc]);
            };
            const bool last_round = r == n_rounds - 1;
            int flushed = 0, ibase = it_round;
            for (int g0 = 0; g0 < n_ang; g0 += 32) {
                const TcBatch bt = tc_batch(g0, n_ang, dX, dY, a);
                for (int i = grp; i < bt.n; i += kG) {
                    const int ab = a.a0 + g0 + i;
                    // flush the blocks that ended kLag angles ago: this group's slot waits proved
                    // their MMAs retired, so the accfull waits return at once
                    PROBE_T0(q3);
                    while (flushed < n_blk && (blk0 + flushed + 1) * kP + kLag <= ab) flush(flushed++);
                    PROBE_ADD(p_flush, q3);
                    const TcWin w = tc_bcast(bt.w, i);
                    const int nk = 1 + ((bt.two >> i) & 1);
                    const int it0 = ibase + i + __popc(bt.two & ((1u << i) - 1u));
#ifdef TF_TC_PROBE_W_IDLE  // probe builds only: no weight arithmetic
                    const float t = 0.f;
#else
                    const float t = fmaxf(fmaf(fdy, w.C, fmaf(fdx, w.B, w.F0)), 0.f);
#endif
                    const float fl = floorf(t);
                    const float f = t - fl;
                    const float g0w = 1.f - f;
                    const __half h0 = __float2half_rn(g0w), h1 = __float2half_rn(f);
                    const __half l0 = __float2half_rn(g0w - __half2float(h0)), l1 = __float2half_rn(f - __half2float(h1));
                    const __half z = __ushort_as_half(0);
                    const int o0 = (int)fl;
                    const bool odd = o0 & 1;
                    const uint32_t Xh = odd ? pack_h2(z, h0) : pack_h2(h0, h1), Yh = odd ? pack_h2(h1, z) : 0u;
                    const uint32_t Xl = odd ? pack_h2(z, l0) : pack_h2(l0, l1), Yl = odd ? pack_h2(l1, z) : 0u;
                    for (int ks = 0; ks < nk; ++ks) {
                        const int it = it0 + ks, s = it % kS;
                        // tap o = floor(t) - 16 ks of this item's window; the pair (2j, 2j + 1) of
                        // halves holding it is jo = o >> 1 (o = -1: only f lands, in pair 0)
                        const int jo = real ? (o0 - kK * ks) >> 1 : -8;
                        PROBE_T0(q4);
                        if (it >= kS) mbar_wait(&empty[s], (uint32_t)((it / kS) - 1) & 1u);
                        PROBE_ADD(p_empty, q4);
                        if (q == 0 && lane == 0) {
                            // this item's taps (the group's lane-quadrant-0 warp issues them as soon as
                            // the slot is free) and the MMA warp's control word: accumulate = 0 (block's
                            // first item), commit the block (its last), accumulator, end of the CTA's
                            // work, wait for the accumulator's flush (from the third block on) and that
                            // wait's phase
                            const int g = ab - a.a0, gb = blk_round + ab / kP - blk0;
                            const bool first = ks == 0 && (g == 0 || ab % kP == 0);
                            const bool last = ks == nk - 1 && (g == n_ang - 1 || (ab + 1) % kP == 0);
                            s_ctl[s] = (first ? 1u : 0u) | (last ? 2u : 0u) | ((uint32_t)(gb & 1) << 2) |
                                       ((last_round && ks == nk - 1 && g == n_ang - 1) ? 8u : 0u) |
                                       ((first && gb >= 2) ? 16u : 0u) | ((uint32_t)(((gb >> 1) - 1) & 1) << 5);
                            uint8_t* st = ring + s * Cfg::SLOT;
                            const int ka = 2 * (ab - a.ws_a0);
#ifdef TF_TC_PROBE_NO_TMA  // probe builds only: timing without the tap loads
                            mbar_arrive(&full[s]);
                            (void)st, (void)ka;
#else
                            mbar_arrive_expect_tx(&full[s], 2 * Cfg::TAP_PLANE);
                            // one box holds both planes (T_hi, T_lo are adjacent along the map's dim 2)
                            tma_load_3d(st, &map, &full[s], 8 * (w.c_lo + kK * ks), zr0 / 8, ka);
#endif

                        }
                        const uint32_t wa = wslot0 + (uint32_t)(s * Cfg::SLOT);
#pragma unroll
                        for (int c = 0; c < 2; ++c) {  // 8-channel chunk c: pairs 4c .. 4c + 3
                            uint32_t vh[4], vl[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const int jj = 4 * c + j;
                                vh[j] = jj == jo ? Xh : (jj == jo + 1 ? Yh : 0u);
                                vl[j] = jj == jo ? Xl : (jj == jo + 1 ? Yl : 0u);
                            }
#ifndef TF_TC_PROBE_NO_WEIGHTS  // probe builds only: timing without the weight stores
                            sts128(wa + 128 * c, vh[0], vh[1], vh[2], vh[3]);
                            sts128(wa + kWPlane + 128 * c, vl[0], vl[1], vl[2], vl[3]);
#else
                            if (vh[0] == 0x7fffffffu && vl[3] == 0x7fffffffu) sts128(wa, vh[0], vh[1], vh[2], vh[3]);
#endif
                        }
#ifndef TF_TC_PROBE_NO_FENCE  // probe builds only
                        fence_proxy_async();  // generic-proxy stores -> visible to the tensor core
#endif
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&full[s]);
                    }
                }
                ibase += bt.n + __popc(bt.two);
            }
            PROBE_T0(q5);
            while (flushed < n_blk) flush(flushed++);
            it_round = ibase;
            blk_round += n_blk;
            // ---- epilogue: master x 2^-e -> volume (fbp.py:247-251)
            int x, y;
            if (voxel(x, y)) {
                const int zc0 = zr0 + grp * NC;  // first volume row of this thread's master columns
                const bool fin = (a.flags & TF_BP_FINALIZE) != 0;
                const bool zero = fin && tc_outside_fov(x, y, a);
                float* out = a.vol + (size_t)y * a.nx + x;
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    const int zz = zc0 + j;
                    if (zz < a.n_rows) {
                        float val = master[j] * s_dn[grp * NC + j];
                        if (fin) val = zero ? 0.f : val * a.angle_wf;
                        out[(size_t)zz * plane] = val;
                    }
                }
            }
            // ---- lockstep: the next round starts when every CTA has finished this one.  Every CTA
            // counts every round it ran; a CTA with a next round waits for all G of this round (all G
            // ran round r whenever any CTA has a round r + 1).  A wait far beyond any round's length
            // means a CTA was never scheduled: trap instead of hanging.
            named_bar_sync(1, 128 * kG);
            if (threadIdx.x == 64) {
                __threadfence();
                atomicAdd(a.sync, 1u);
#ifndef TF_TC_PROBE_NO_LOCKSTEP  // probe builds only: rounds without the grid barrier
                if (!last_round) {
#else
                if (false) {
#endif
                    const unsigned target = (unsigned)(r + 1) * (unsigned)G;
                    const long long t0 = clock64();
                    while (*reinterpret_cast<volatile unsigned*>(a.sync) < target) {
                        __nanosleep(64);
                        if (clock64() - t0 > 20000000000LL) __trap();
                    }
                    __threadfence();
                }
            }
            PROBE_ADD(p_tail, q5);
        }
#ifdef TF_TC_PROBE
        if (a.probe && lane == 0 && blockIdx.x < 1024 && warp == 2) a.probe[blockIdx.x * 16 + 13] = p_tail;
        if (a.probe && lane == 0 && blockIdx.x < 1024 && (warp == 2 || warp == 14)) {
            const int o = warp == 2 ? 7 : 10;
            a.probe[blockIdx.x * 16 + o] = clock64() - p_start;
            a.probe[blockIdx.x * 16 + o + 1] = p_empty;
            a.probe[blockIdx.x * 16 + o + 2] = p_flush;
        }
#endif
        (void)p_empty, (void)p_flush, (void)p_tail;
    }
#ifdef TF_TC_PROBE_W_NONE
probe_done:
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::TMEM_COLS));
}

// FINALIZE over the tiles wholly outside the field of view (not in the persistent kernel's work
// list): zeros inside the requested tile (fbp.py:247-250 masks them)
__global__ void tc_zero_tiles_kernel(float* __restrict__ vol, const int* __restrict__ tiles, int n_tiles, int ntx,
                                     int nx, int ny, int n_rows, int x0, int x1, int y0, int y1) {
    const long long per = (long long)kMV * n_rows;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n_tiles * per;
         i += (long long)gridDim.x * blockDim.x) {
        const int t = tiles[i / per];
        const long long r = i % per;
        const int z = (int)(r / kMV), v = (int)(r % kMV);
        const int x = (t % ntx) * kTX + v % kTX, y = (t / ntx) * kTY + v / kTX;
        if (x >= x0 && x < x1 && y >= y0 && y < y1 && x < nx && y < ny) vol[((size_t)z * ny + y) * nx + x] = 0.f;
    }
}

// ---- tap planes from natural-layout filtered rows (the fbp.back_project input) -------------
// Per-row max |T w| over the angles and channels (non-negative floats order as their bits).
__global__ void tc_rowmax_kernel(const float* __restrict__ sino, const float* __restrict__ w, int rows_per_angle,
                                 int r0, int k, int a0, int n_ang, int n_chan, unsigned* __restrict__ mx) {
    const int lane = threadIdx.x & 31;
    const long long n_lines = (long long)n_ang * k;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long l = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); l < n_lines; l += warps) {
        const int r = (int)(l % k);
        const long long ang = a0 + l / k;
        const float* src = sino + ((size_t)ang * rows_per_angle + r0 + r) * n_chan;
        float v = 0.f;
        for (int c = lane; c < n_chan; c += 32) {
            const float e = fabsf(src[c] * (w ? w[c] : 1.f));
            if (e <= 3.0e38f) v = fmaxf(v, e);  // inf / nan do not set the scale
        }
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0 && v > 0.f) atomicMax(&mx[r], __float_as_uint(v));
    }
}

// e = 14 - ilogb(bound): bound x 2^e in [2^14, 2^15), clamped so 2^(+-e) stays a normal float
__device__ __forceinline__ int tap_exponent(float bound) {
    return bound > 0.f ? min(100, max(-100, 14 - ilogbf(bound))) : 0;
}

// e[r] from a uniform bound (> 0) or from the row maxima x factor
__global__ void tc_exponent_kernel(const unsigned* __restrict__ mx, int* __restrict__ e, int k, float bound,
                                   float factor) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k; r += gridDim.x * blockDim.x)
        e[r] = tap_exponent(bound > 0.f ? bound : __uint_as_float(mx[r]) * factor);
}

// fp16 hi/lo split of x (|x| < 2^15 by the exponent; saturated so an undersized caller bound
// gives wrong values, never inf/nan that the zero weights would spread over the tile)
__device__ __forceinline__ void split_h(float x, __half& hi, __half& lo) {
    x = fminf(fmaxf(x, -65504.f), 65504.f);
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}

// natural rows [a][r0 + r][c] -> tap planes [a - a0][hi, lo][r / 8][c][r % 8], feathered
// (fbp.py:242, fp32 product) and scaled by 2^e[r]; one item = 8 rows of one channel
__global__ void tc_stage_kernel(const float* __restrict__ sino, const float* __restrict__ w, int rows_per_angle,
                                int r0, int k, int a0, int n_ang, int n_chan, const int* __restrict__ e,
                                __half* __restrict__ taps) {
    const int R8 = (k + 7) / 8;
    const long long n_items = (long long)n_ang * R8 * n_chan;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_items;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % n_chan);
        const long long rest = i / n_chan;
        const int g8 = (int)(rest % R8);
        const long long ang = rest / R8;
        const float wc = w ? w[c] : 1.f;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __half h[2], l[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int r = g8 * 8 + 2 * j + u;
                float v = 0.f;
                if (r < k) {
                    v = __ldcs(sino + ((size_t)(a0 + ang) * rows_per_angle + r0 + r) * n_chan + c) * wc;
                    v *= __int_as_float((127 + e[r]) << 23);  // x 2^e, exact
                }
                split_h(v, h[u], l[u]);
            }
            hw[j] = pack_h2(h[0], h[1]);
            lw[j] = pack_h2(l[0], l[1]);
        }
        const size_t plane8 = (size_t)R8 * n_chan * 8;  // halves per plane per angle
        __half* dh = taps + (size_t)ang * 2 * plane8 + ((size_t)g8 * n_chan + c) * 8;
        *reinterpret_cast<uint4*>(dh) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dh + plane8) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// Items (MMA K-steps) a launch issues: the same window test as bp_tc_kernel, per FoV-active tile
// and angle (one block per tile; every z-block issues the same items).
__global__ void tc_work_kernel(TCArgs a, int n_active, unsigned long long* __restrict__ out) {
    const int tile = a.tiles[blockIdx.x];
    const int X0 = (tile % a.ntx) * kTX, Y0 = (tile / a.ntx) * kTY;
    const double dX = (double)X0 - a.cx, dY = (double)Y0 - a.cy;
    unsigned long long n = 0;
    for (int g = threadIdx.x; g < a.a1 - a.a0; g += blockDim.x)
        n += 1 + (tc_two_items(tc_window(dX, dY, a.trig[a.a0 + g], a)) ? 1 : 0);
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, n);
}

// ---- workspace geometry ----------------------------------------------------------------------
// [header: int32 e[n_rows] | uint32 rowmax[n_rows] | grid-barrier counter (64 B) | int32 tile list of a
//  restricted call (one per tile of the plane), padded to 1 KB][taps: angle-major planes]
int64_t tc_header_bytes(const tf_bp_plan* p, int n_rows) {
    return ((int64_t)8 * n_rows + 64 + 4 * (int64_t)p->n_tiles[kShapeTc] + 1023) / 1024 * 1024;
}
int64_t tc_angle_bytes(const tf_bp_plan* p, int n_rows) {
    return (int64_t)2 * ((n_rows + 7) / 8) * p->g.n_chan * 16;
}
int* tc_exp_ptr(void* ws) { return static_cast<int*>(ws); }
unsigned* tc_max_ptr(void* ws, int n_rows) { return reinterpret_cast<unsigned*>(static_cast<int*>(ws) + n_rows); }
unsigned* tc_sync_ptr(void* ws, int n_rows) { return reinterpret_cast<unsigned*>(static_cast<int*>(ws) + 2 * n_rows); }
int* tc_tiles_ptr(void* ws, int n_rows) { return static_cast<int*>(ws) + 2 * n_rows + 16; }
__half* tc_taps_ptr(const tf_bp_plan* p, void* ws, int n_rows) {
    return reinterpret_cast<__half*>(static_cast<uint8_t*>(ws) + tc_header_bytes(p, n_rows));
}

TCArgs make_args(const tf_bp_plan* p) {
    TCArgs a{};
    a.trig = p->d_trig;
    a.nx = p->g.nx;
    a.ny = p->g.ny;
    a.ntx = (p->g.nx + kTX - 1) / kTX;
    a.cx = p->cx;
    a.cy = p->cy;
    a.scale = p->scale;
    a.axis = p->axis;
    a.R2 = p->R2;
    a.sc2 = p->sc2;
    a.angle_wf = p->angle_wf;
    return a;
}

template <int NR>
int launch_tc(const CUtensorMap& map, const TCArgs& a, cudaStream_t s) {
    auto* fn = bp_tc_kernel<NR>;
    TF_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<NR>::SMEM));
    int dev = 0, sms = 0, per_sm = 0;
    TF_CUDA_TRY(cudaGetDevice(&dev));
    TF_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, TcCfg<NR>::SMEM));
    if (per_sm < 1) return set_error(TF_ERR_UNSUPPORTED, "bp_tc_kernel does not fit on an SM");
    // every CTA of a round must be resident for the lockstep barrier: a cooperative launch
    const unsigned grid = (unsigned)std::min<long long>((long long)sms * per_sm, a.n_work);
    TCArgs args = a;
    CUtensorMap m = map;
    void* kargs[] = {&m, &args};
    TF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kThreads), kargs, TcCfg<NR>::SMEM, s));
    return check_launch("bp_tc_kernel");
}

}  // namespace

#ifdef TF_TC_PROBE
long long* g_tc_probe = nullptr;  // set by tools/tc_probe.cu's tf_bp_tc_probe (probe build only)
#endif

// shared with filter.cu (K1 writing tap planes directly)
int64_t bp_tc_header_bytes(const tf_bp_plan* p, int n_rows) { return tc_header_bytes(p, n_rows); }
int tc_uniform_exponents(void* taps, int n_rows, double bound, cudaStream_t s) {
    tc_exponent_kernel<<<(n_rows + 255) / 256, 256, 0, s>>>(nullptr, tc_exp_ptr(taps), n_rows, (float)bound, 1.f);
    return check_launch("tc_exponent_kernel");
}
int tc_row_exponents(void* taps, const float* lines, int rows_per_angle, int n_ang, int n_chan, const float* w,
                     double factor, cudaStream_t s) {
    const int k = rows_per_angle;
    TF_CUDA_TRY(cudaMemsetAsync(tc_max_ptr(taps, k), 0, sizeof(unsigned) * k, s));
    if (n_ang > 0) {
        const long long n_lines = (long long)n_ang * k;
        const int grid = (int)std::min<long long>((n_lines + 7) / 8, 148LL * 8);
        tc_rowmax_kernel<<<grid, 256, 0, s>>>(lines, w, rows_per_angle, 0, k, 0, n_ang, n_chan, tc_max_ptr(taps, k));
    }
    tc_exponent_kernel<<<(k + 255) / 256, 256, 0, s>>>(tc_max_ptr(taps, k), tc_exp_ptr(taps), k, 0.f,
                                                       (float)factor);
    return check_launch("tc_exponent_kernel");
}
}  // namespace tf

using namespace tf;

extern "C" int tf_bp_tc_supported(const tf_bp_plan* p) {
    // an 11 x 11 tile's rays span <= 10 sqrt(2) scale + 2 taps; two items hold 32 channels
    return p && 10.0 * std::sqrt(2.0) * p->scale + 2.0 <= 2.0 * kK ? 1 : 0;
}

extern "C" int64_t tf_bp_tc_taps_bytes(const tf_bp_plan* p, int n_rows, int n_angles) {
    if (!p || n_rows < 0 || n_angles < 0) return -1;
    return tc_header_bytes(p, n_rows) + (int64_t)n_angles * tc_angle_bytes(p, n_rows);
}

extern "C" int tf_bp_tc_set_exponent(const tf_bp_plan* p, void* taps, int n_rows, double t_bound, void* stream) {
    if (!p || !taps) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    if (n_rows <= 0) return n_rows == 0 ? TF_OK : set_error(TF_ERR_INVALID_ARGUMENT, "n_rows must be >= 0");
    if (!(t_bound > 0)) return set_error(TF_ERR_INVALID_ARGUMENT, "t_bound must be positive");
    return tc_uniform_exponents(taps, n_rows, t_bound, as_stream(stream));
}

extern "C" int tf_bp_tc_stage(const tf_bp_plan* p, const float* sino, int rows_per_angle, int r0, int r1, int a0,
                              int a1, double t_bound, void* taps, int64_t taps_bytes, void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null bp plan");
    if (!tf_bp_tc_supported(p))
        return set_error(TF_ERR_UNSUPPORTED, "tensor-core back-projection needs voxel_pitch / pixel_pitch <= %.3f",
                         (2.0 * kK - 2.0) / (10.0 * std::sqrt(2.0)));
    if (!(0 <= r0 && r0 <= r1 && r1 <= rows_per_angle))
        return set_error(TF_ERR_INVALID_ARGUMENT, "row range (%d, %d) out of bounds", r0, r1);
    if (!(0 <= a0 && a0 <= a1 && a1 <= p->g.n_proj))
        return set_error(TF_ERR_INVALID_ARGUMENT, "angle range (%d, %d) out of bounds", a0, a1);
    const int k = r1 - r0;
    if (k == 0) return TF_OK;
    if (!sino || !taps) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    if (taps_bytes < tf_bp_tc_taps_bytes(p, k, a1 - a0))
        return set_error(TF_ERR_INVALID_ARGUMENT, "tap workspace too small: %lld < %lld bytes", (long long)taps_bytes,
                         (long long)tf_bp_tc_taps_bytes(p, k, a1 - a0));
    cudaStream_t s = as_stream(stream);
    const float* w = p->g.scan_mode ? p->d_w : nullptr;
    if (t_bound > 0) {
        int st = tc_uniform_exponents(taps, k, t_bound, s);
        if (st) return st;
    } else {  // per-row scale from the data (all angles of the call)
        TF_CUDA_TRY(cudaMemsetAsync(tc_max_ptr(taps, k), 0, sizeof(unsigned) * k, s));
        if (a1 > a0) {
            const long long lines = (long long)(a1 - a0) * k;
            const int grid = (int)std::min<long long>((lines + 7) / 8, 148LL * 8);
            tc_rowmax_kernel<<<grid, 256, 0, s>>>(sino, w, rows_per_angle, r0, k, a0, a1 - a0, p->g.n_chan,
                                                  tc_max_ptr(taps, k));
        }
        tc_exponent_kernel<<<(k + 255) / 256, 256, 0, s>>>(tc_max_ptr(taps, k), tc_exp_ptr(taps), k, 0.f, 1.f);
    }
    if (a1 > a0) {
        const long long items = (long long)(a1 - a0) * ((k + 7) / 8) * p->g.n_chan;
        const int grid = (int)std::min<long long>((items + 255) / 256, 148LL * 16);
        tc_stage_kernel<<<grid, 256, 0, s>>>(sino, w, rows_per_angle, r0, k, a0, a1 - a0, p->g.n_chan,
                                             tc_exp_ptr(taps), tc_taps_ptr(p, taps, k));
    }
    return check_launch("tc_stage_kernel");
}

extern "C" int tf_backproject_tc(const tf_bp_plan* p, const void* taps, int64_t taps_bytes, int taps_a0,
                                 int taps_a1, int n_rows, float* vol, int a0, int a1, int x0, int x1, int y0, int y1,
                                 int flags, void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null bp plan");
    const tf_geometry& g = p->g;
    if (!tf_bp_tc_supported(p))
        return set_error(TF_ERR_UNSUPPORTED, "tensor-core back-projection needs voxel_pitch / pixel_pitch <= %.3f",
                         (2.0 * kK - 2.0) / (10.0 * std::sqrt(2.0)));
    if (!(0 <= taps_a0 && taps_a0 <= a0 && a0 <= a1 && a1 <= taps_a1 && taps_a1 <= g.n_proj))
        return set_error(TF_ERR_INVALID_ARGUMENT, "angle range (%d, %d) outside the staged (%d, %d)", a0, a1, taps_a0,
                         taps_a1);
    if (!(0 <= x0 && x0 <= x1 && x1 <= g.nx && 0 <= y0 && y0 <= y1 && y1 <= g.ny))
        return set_error(TF_ERR_INVALID_ARGUMENT, "tile (%d, %d, %d, %d) out of bounds", x0, x1, y0, y1);
    if (n_rows < 0) return set_error(TF_ERR_INVALID_ARGUMENT, "n_rows must be >= 0");
    if (n_rows == 0 || x0 == x1 || y0 == y1) return TF_OK;
    if (!taps || !vol) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    if (taps_bytes < tf_bp_tc_taps_bytes(p, n_rows, taps_a1 - taps_a0))
        return set_error(TF_ERR_INVALID_ARGUMENT, "tap workspace too small: %lld < %lld bytes", (long long)taps_bytes,
                         (long long)tf_bp_tc_taps_bytes(p, n_rows, taps_a1 - taps_a0));
    const int R8 = (n_rows + 7) / 8;
    const int NR = n_rows > 128 ? 256 : 128;

    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    CUtensorMap map;
    void* ws = const_cast<void*>(taps);
    void* data = tc_taps_ptr(p, ws, n_rows);
    // dim 0 = (channel, row-in-group) flattened: a box row is 16 channels x 8 rows = 256 contiguous
    // bytes; channel c starts at element 8 c.  dim 1 = 8-row group, dim 2 = (angle, plane).
    cuuint64_t dims[3] = {(cuuint64_t)8 * g.n_chan, (cuuint64_t)R8, (cuuint64_t)(2 * (taps_a1 - taps_a0))};
    cuuint64_t strides[2] = {(cuuint64_t)g.n_chan * 16u, (cuuint64_t)R8 * g.n_chan * 16u};
    cuuint32_t box[3] = {(cuuint32_t)(8 * kK), (cuuint32_t)(NR / 8), 2u};  // T_hi and T_lo of one step
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, data, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    cudaStream_t s = as_stream(stream);

    TCArgs a = make_args(p);
    a.e_rows = tc_exp_ptr(ws);
    a.sync = tc_sync_ptr(ws, n_rows);
    a.vol = vol;
    a.a0 = a0;
    a.a1 = a1;
    a.ws_a0 = taps_a0;
    a.n_rows = n_rows;
    a.x0 = x0;
    a.x1 = x1;
    a.y0 = y0;
    a.y1 = y1;
    a.flags = flags & (TF_BP_ACCUMULATE | TF_BP_FINALIZE);
#ifdef TF_TC_PROBE
    a.probe = g_tc_probe;
#endif
    // the work list: the FoV-active tiles of the plan (Morton order), or of them the ones overlapping
    // a restricted tile -- copied into the workspace header
    const int n_act = p->n_active[kShapeTc];
    if (x0 == 0 && x1 == g.nx && y0 == 0 && y1 == g.ny) {
        a.tiles = p->d_order[kShapeTc];
        a.n_tiles = n_act;
    } else {
        std::vector<int> sel;
        for (int i = 0; i < n_act; ++i) {
            const int t = p->h_order[kShapeTc][i];
            const int X0 = (t % a.ntx) * kTX, Y0 = (t / a.ntx) * kTY;
            if (X0 < x1 && X0 + kTX > x0 && Y0 < y1 && Y0 + kTY > y0) sel.push_back(t);
        }
        if (!sel.empty())
            TF_CUDA_TRY(cudaMemcpyAsync(tc_tiles_ptr(ws, n_rows), sel.data(), sizeof(int) * sel.size(),
                                        cudaMemcpyHostToDevice, s));
        a.tiles = tc_tiles_ptr(ws, n_rows);
        a.n_tiles = (int)sel.size();
    }
    a.n_work = a.n_tiles * ((n_rows + NR - 1) / NR);
    if (a.flags & TF_BP_FINALIZE) {  // the FoV-inactive tiles are only masked: zeros
        const int n_in = p->n_tiles[kShapeTc] - n_act;
        if (n_in > 0) {
            const long long n = (long long)n_in * kMV * n_rows;
            const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
            tc_zero_tiles_kernel<<<grid, 256, 0, s>>>(vol, p->d_order[kShapeTc] + n_act, n_in, a.ntx, g.nx, g.ny, n_rows,
                                                      x0, x1, y0, y1);
            int st = check_launch("tc_zero_tiles_kernel");
            if (st) return st;
        }
    }
    if (a.n_work == 0) return TF_OK;
    TF_CUDA_TRY(cudaMemsetAsync(a.sync, 0, sizeof(unsigned), s));
    return NR == 256 ? launch_tc<256>(map, a, s) : launch_tc<128>(map, a, s);
}

extern "C" int tf_bp_tc_work(const tf_bp_plan* p, int n_rows, int a0, int a1, int64_t* items,
                             int64_t* executed_updates, int64_t* mma_clocks) {
    if (!p || !items || !executed_updates || !mma_clocks) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    if (!(0 <= a0 && a0 <= a1 && a1 <= p->g.n_proj) || n_rows < 0)
        return set_error(TF_ERR_INVALID_ARGUMENT, "invalid rows/angles");
    const int NR = n_rows > 128 ? 256 : 128;
    const int64_t zblocks = (n_rows + NR - 1) / NR;
    unsigned long long per_zblock = 0;
    const int na = p->n_active[kShapeTc];
    if (na > 0 && a1 > a0 && n_rows > 0) {
        unsigned long long* d = nullptr;
        TF_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long)));
        cudaError_t e = cudaMemset(d, 0, sizeof(unsigned long long));
        TCArgs a = make_args(p);
        a.a0 = a0;
        a.a1 = a1;
        a.tiles = p->d_order[kShapeTc];
        if (e == cudaSuccess) {
            tc_work_kernel<<<na, 256>>>(a, na, d);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpy(&per_zblock, d, sizeof(per_zblock), cudaMemcpyDeviceToHost);
        cudaFree(d);
        if (e != cudaSuccess) return set_error(TF_ERR_CUDA, "tc work count failed: %s", cudaGetErrorString(e));
    }
    // voxel x angle x row updates of the active tiles (tile voxels inside the volume)
    int64_t vox = 0;
    {
        const int ntx = (p->g.nx + kTX - 1) / kTX;
        std::vector<int> order(na);
        if (na > 0) TF_CUDA_TRY(cudaMemcpy(order.data(), p->d_order[kShapeTc], sizeof(int) * na, cudaMemcpyDeviceToHost));
        for (int t : order) {
            const int X0 = (t % ntx) * kTX, Y0 = (t / ntx) * kTY;
            vox += (int64_t)(std::min(X0 + kTX, p->g.nx) - X0) * (std::min(Y0 + kTY, p->g.ny) - Y0);
        }
    }
    *items = (int64_t)per_zblock * zblocks;
    *executed_updates = vox * (int64_t)n_rows * (a1 - a0);
    *mma_clocks = *items * 3 * (NR / 2);  // 3 MMAs of 128 x NR x 16 per item at NR / 2 clk each
    return TF_OK;
}

// EXPERIMENT (not the product kernel): K2-TC with the weights as the TMEM A operand and
// 4-step items, measured against paper_2505_13955_b200/csrc/bp_tc.cu and not kept
// ("Where the time goes").  Parity-green (37 tensor-path GPU tests) but
// 21% slower at C3 rows: 674 ms per 1152 rows vs 496 ms per 1024 rows.  A/B timing:
//     python tools/tc_probe.py --build --define TF_TC_NOPROBE --src tools/micro/bp_tc_tmem_items.cu
//
// K2-TC: back-projection on the 5th-generation tensor cores (tcgen05).
// Replaces fbp.back_project (fbp.py:186-252) on the default path.
//
// For one angle, a tile of 121 voxel columns (11 x 11, padded to the MMA's
// M = 128) and N detector rows, back-projection is a small GEMM
//     D[m][z] += sum_k W[m][k] * T[k][z],
// T the feathered filtered taps of the tile's channel window [c_lo, c_lo+16)
// and W the interpolation matrix: row m holds voxel m's exact two-tap weights
// {1 - f, f} at k = floor(t) - c_lo and k + 1, zeros elsewhere
// (fbp.py:237-245).  Summed over the angles, D is the unscaled
// back-projection.  The tile's window spans 10 (|cos| + |sin|) + 1 <= 15.2
// channels, so 97% of the angles need one K = 16 "step"; the others need two
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
// Hand-offs are the budget: measured with the MMAs, the tap loads and the
// weight stores all compiled out, one barrier round trip per K-step cost
// ~460 clk -- more than the step's 3 MMAs (288 clk at N = 192).  So the unit
// of synchronisation is an ITEM of kQ = 4 consecutive steps (one slot wait,
// one arrival per warp, one commit per item), and the weights live in
// tensor memory (tcgen05.st by the weight warps, the MMAs read A from TMEM),
// so shared memory carries only the taps.
//
// CTA (576 threads, one per SM), TMEM = two ping-pong accumulators of
// kNB = 192 columns + a 2-item ring of A tiles (4 steps x 16 columns each):
//   warp 0      TMA producer: the fp64 window origin per angle and one
//               cp.async.bulk.tensor box per step (T_hi and T_lo: 16 channels
//               x N rows x 2 planes, MN-major canonical layout) into a
//               4-item ring; the OOB zero fill is the reference's zero guard
//               for off-detector taps;
//   warp 1      TMEM owner and MMA issuer: per step, one elected lane issues
//               3 tcgen05.mma.kind::f16 (A = W from TMEM, B = T from shared
//               memory); one commit per item frees its tap and A slots;
//   warps 2-17  four weight groups of 4 warps (step j of every item -> group
//               j; one voxel row per thread = one TMEM lane): fp32 t relative
//               to the fp64 window origin, the fp16 hi/lo W row of the step,
//               and its control word for the MMA warp.  Every warp
//               also owns N/4 columns of the RN master sum of its 32 voxels
//               (<= 48 registers): it flushes each finished block as soon as
//               its MMAs retire -- polled while it waits for an A slot --
//               (tcgen05.ld + fadd.rn) and writes the epilogue (x 2^-e, FoV
//               mask and angle weight, fbp.py:247-251).
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
constexpr int kK = 16;          // channels per step (one fp16 MMA K-step)
constexpr int kNB = 192;        // rows of a z-block at most (MMA N)
constexpr int kQ = 4;           // steps per item
constexpr int kSi = 4;          // tap ring depth in items
constexpr int kAi = 2;          // A ring depth in items (TMEM)
constexpr int kP = 16;          // angles per accumulator block (absolute angle index / kP)
constexpr int kG = 4;           // weight groups of 4 warps
constexpr int kThreads = 64 + 128 * kG;
// completion barriers: done[i % kB] completes when item i's MMAs retire.  A parity wait is only
// unambiguous within one phase: the TMA warp and every weight warp wait for the items in order
constexpr int kB = 4;
static_assert(kQ == kG && (kQ & (kQ - 1)) == 0, "step j of an item is group j's");
constexpr int kStep = 2 * kNB * kK * 2;    // one step's taps in shared memory: hi, lo planes (12 KB)
constexpr int kSlot = kQ * kStep;          // one item's taps (48 KB)
constexpr int kNC = kNB / kG;              // master columns per thread (at most)
constexpr uint32_t kAcol = 2 * kNB;        // first TMEM column of the A ring
constexpr uint32_t kAslot = kQ * 16;       // TMEM columns per A slot (hi at +0, lo at +8 per step)
constexpr uint32_t kTmemCols = 512;
constexpr int kSmem = kSi * kSlot + kNB * 8 + (kSi + kAi + kB + 4) * 8 + 16 + 4 * kAi * (kQ + 1);
constexpr float kOneStep = 14.9f;          // window test (fp32 margin below 15)
static_assert(kMV <= kM, "tile fits the MMA's M");
static_assert(kAcol + kAslot * kAi <= kTmemCols, "accumulators + A ring fit TMEM");
static_assert(kNB % 32 == 0 && kNC % 8 == 0, "column slices");
static_assert(kSlot % 1024 == 0 && kStep % 128 == 0, "TMA destinations stay aligned");
static_assert(32 % kG == 0, "a batch of 32 angles splits evenly over the groups");

// D f32, A f16 K-major, B f16 MN-major, M = 128; N (bits 17-22, N >> 3) per z-block
constexpr uint32_t kIdesc = (1u << 4) | (1u << 16) | ((uint32_t)(kM >> 4) << 24);

// per-step control word (written by the producing group, read by the MMA warp)
constexpr uint32_t kCtlFirst = 1u;     // the block's first step: accumulate = 0
constexpr uint32_t kCtlLast = 2u;      // the block's last step: commit accfull after it
constexpr uint32_t kCtlAcc = 4u;       // accumulator index
constexpr uint32_t kCtlFree = 16u;     // wait for the accumulator's previous block to be flushed
constexpr uint32_t kCtlFreePh = 32u;   // ... that wait's phase
constexpr int kCtlN = 8;               // N / 16 at bit 8
// per-item count word: steps in the item, and the end of the CTA's work
constexpr uint32_t kCntEnd = 256u;

struct TCArgs {
    const double2* trig;
    const int* tiles;   // work list: FoV-active tiles (Morton order) of one z-block
    int n_tiles, n_work;  // tiles per z-block; work items = z-blocks x n_tiles
    unsigned* sync;     // grid-barrier counter of the lockstep rounds (workspace header, zeroed per call)
    const int* e_rows;  // per-row tap exponent (workspace header)
    float* vol;
    int a0, a1, ws_a0, n_rows, nx, ny;
    int nb, nzb, n_last, tx_bytes;  // z-block rows, z-blocks, the last block's N, TMA bytes per step
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

// D (TMEM) (+)= A (TMEM) x B (shared memory descriptor)
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc)
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

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
    return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
}

#define TC_LD8(ta, v)                                                                                   \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"               \
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), \
                   "=r"(v[7])                                                                           \
                 : "r"(ta))

#define TC_ST16(ta, v)                                                                                          \
    asm volatile(                                                                                               \
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
        ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),     \
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])           \
        : "memory")

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
// one step when every tap of the tile lies in the window's first 16 channels
__device__ __forceinline__ bool tc_two_steps(const TcWin& w) {
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
// of the angles that need two steps (every role walks the same step sequence)
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
    b.two = __ballot_sync(0xffffffffu, g0 + lane < n_ang && tc_two_steps(b.w));
    b.n = min(32, n_ang - g0);
    return b;
}

__device__ __forceinline__ bool tc_outside_fov(int x, int y, const TCArgs& a) {
    // ((x-cx)^2 + (y-cy)^2) * scale^2 > R^2, no FMA contraction (fbp.py:247-250)
    double dx = __dsub_rn((double)x, a.cx), dy = __dsub_rn((double)y, a.cy);
    double rr = __dmul_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), a.sc2);
    return rr > a.R2;
}

// non-suspending barrier poll (mbarrier.test_wait): try_wait may park the warp for a
// hardware-defined time, which on a tight hand-off chain costs more than the work
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
    while (!mbar_test(bar, parity)) {
    }
}
#ifdef TF_TC_SPIN_MMA
#define tc_wait_mma(bar, parity) mbar_spin(bar, parity)
#else
#define tc_wait_mma(bar, parity) mbar_wait(bar, parity)
#endif
#ifdef TF_TC_SPIN_W
#define tc_poll_w(bar, parity) mbar_test(bar, parity)
#else
#define tc_poll_w(bar, parity) mbar_try_wait(bar, parity)
#endif

#if defined(TF_TC_HANG_DEBUG) && defined(TF_TC_PROBE)
// debug probe builds only: a wait longer than ~0.25 s is recorded (count, smallest item, block,
// thread, parity per wait tag) in the probe buffer's last 64 entries; after ~2 s every wait gives up
__device__ __forceinline__ void tc_wait_dbg(uint64_t* bar, uint32_t parity, int tag, int it, long long* dbg) {
    volatile long long* dead = dbg + 1024 * 16 - 1;
    const long long t0 = clock64();
    bool rec = false;
    while (!mbar_try_wait(bar, parity)) {
        const long long dt = clock64() - t0;
        if (!rec && dt > 500000000LL) {
            rec = true;
            long long* d = dbg + 1024 * 16 - 64 + tag * 8;
            atomicAdd(reinterpret_cast<unsigned long long*>(d), 1ull);
            atomicMin(d + 1, (long long)it);
            d[2] = blockIdx.x;
            d[3] = threadIdx.x;
            d[4] = parity;
        }
        if (dt > 4000000000LL) *dead = 1;
        if (*dead) return;
    }
}
#define tc_wait(bar, parity, tag, it) tc_wait_dbg(bar, parity, tag, it, a.probe)
#else
#define tc_wait(bar, parity, tag, it) mbar_wait(bar, parity)
#endif

// work item wi -> its z-block and tile
struct TcWork {
    int zb, tile, zr0, n;  // z-block, tile, first row, MMA N (rows, multiple of 16)
};
__device__ __forceinline__ TcWork tc_work(int wi, const TCArgs& a) {
    TcWork w;
    w.zb = wi / a.n_tiles;
    w.tile = a.tiles[wi - w.zb * a.n_tiles];
    w.zr0 = w.zb * a.nb;
    w.n = w.zb == a.nzb - 1 ? a.n_last : a.nb;
    return w;
}

// Persistent, lockstep: the grid is one CTA per SM (cooperative launch) and
// CTA b processes the work items w = r G + b (r = 0, 1, ...) of the list of
// (z-block, FoV-active tile) pairs, z-block outer, tiles in Morton order.  A
// grid-wide barrier between rounds keeps the G CTAs of a round -- a compact
// patch of Morton-adjacent tiles -- at the same angle within a few percent,
// so the patch's tap windows are fetched from DRAM once and re-read from L2
// by its other CTAs (a grid of one CTA per tile let resident CTAs sit at
// unrelated angles: 2.4 TB of DRAM reads per C3 volume, 62% L2 hits).  The
// rings, their phases and the accumulator ping-pong run on across the
// rounds; a round's steps are packed into items of kQ (its last item may be
// shorter, so no item spans a round), each round resets the RN master sum
// and ends with the epilogue.
__global__ void __launch_bounds__(kThreads, 1) bp_tc_kernel(const __grid_constant__ CUtensorMap map, const TCArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const size_t plane = (size_t)a.nx * a.ny;
    const int G = gridDim.x;
    const int n_rounds = a.n_work > (int)blockIdx.x ? (a.n_work - 1 - (int)blockIdx.x) / G + 1 : 0;

    uint8_t* const ring = smem;  // [kSi] tap slots: [kQ] steps of T_hi, T_lo
    float* s_up = reinterpret_cast<float*>(ring + kSi * kSlot);  // per row of the round: 2^e and 2^-e
    float* s_dn = s_up + kNB;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_dn + kNB);  // [kSi] an item's taps landed
    uint64_t* afull = full + kSi;     // [kAi] the 16 weight warps stored the item's A tiles
    uint64_t* done = afull + kAi;     // [kB] item i's MMAs retired (done[i % kB]): its slots are free
    uint64_t* accfull = done + kB;    // [2]: block's MMAs done -> flush
    uint64_t* accfree = accfull + 2;  // [2]: block flushed by all 16 weight warps -> accumulator reusable
    uint32_t* tslot = reinterpret_cast<uint32_t*>(accfree + 2);
    uint32_t* s_ctl = tslot + 4;        // [kAi][kQ]: the A slot's step control words
    uint32_t* s_cnt = s_ctl + kAi * kQ;  // [kAi]: steps in the item | kCntEnd
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSi; ++s) mbar_init(&full[s], 1);  // the TMA warp's arrive (+ transaction bytes)
        for (int s = 0; s < kAi; ++s) mbar_init(&afull[s], 4 * kG);  // every weight warp (step j of an item is group j's)
        for (int s = 0; s < kB; ++s) mbar_init(&done[s], 1);    // MMA commit
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accfull[b], 1);
            mbar_init(&accfree[b], 4 * kG);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // columns [0, kNB) accumulator 0, [kNB, 2 kNB) accumulator 1, [kAcol, kAcol + kAi kAslot) the A ring
    const uint32_t tmem = *tslot;
    const int n_ang = a.a1 - a.a0;
    const int blk0 = a.a0 / kP;  // first absolute block
    const int n_blk = n_ang > 0 ? (a.a1 - 1) / kP - blk0 + 1 : 0;

    if (warp == 0) {
        // ---- TMA: walks the same step sequence, up to kSi items ahead of the MMAs
        if (lane == 0) tma_prefetch_desc(&map);
        long long p_wait = 0;
        PROBE_T0(p_start);
        int item = 0;
        for (int r = 0; r < n_rounds && n_ang > 0; ++r) {
            const TcWork wk = tc_work(r * G + (int)blockIdx.x, a);
            const double dX = (double)((wk.tile % a.ntx) * kTX) - a.cx, dY = (double)((wk.tile / a.ntx) * kTY) - a.cy;
            int j = 0;  // step within the current item
            for (int g0 = 0; g0 < n_ang; g0 += 32) {
                const TcBatch bt = tc_batch(g0, n_ang, dX, dY, a);
                for (int i = 0; i < bt.n; ++i) {
                    const int c_lo = __shfl_sync(0xffffffffu, bt.w.c_lo, i);
                    const int nk = 1 + ((bt.two >> i) & 1);
                    const int ka = 2 * (a.a0 + g0 + i - a.ws_a0);
                    if (lane == 0) {
                        for (int ks = 0; ks < nk; ++ks) {
                            const int s = item % kSi;
                            if (j == 0 && item >= kSi) {
                                const int x = item - kSi;  // the slot's previous item
                                PROBE_T0(q0);
                                tc_wait(&done[x % kB], (uint32_t)(x / kB) & 1u, 0, item);
                                PROBE_ADD(p_wait, q0);
                            }
                            uint8_t* st = ring + s * kSlot + j * kStep;
#ifdef TF_TC_PROBE_NO_TMA  // probe builds only: timing without the tap loads
                            (void)st, (void)ka, (void)c_lo;
#else
                            mbar_expect_tx(&full[s], (uint32_t)a.tx_bytes);
                            tma_load_3d(st, &map, &full[s], 8 * (c_lo + kK * ks), wk.zr0 / 8, ka);
#endif
                            if (++j == kQ) {
                                mbar_arrive(&full[s]);
                                j = 0;
                                ++item;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            if (lane == 0 && j) mbar_arrive(&full[item % kSi]);  // the round's last, short item
            item = __shfl_sync(0xffffffffu, item + (j ? 1 : 0), 0);
        }
#ifdef TF_TC_PROBE
        if (a.probe && lane == 0 && blockIdx.x < 1024) {
            a.probe[blockIdx.x * 16 + 0] = clock64() - p_start;
            a.probe[blockIdx.x * 16 + 1] = p_wait;
        }
#endif
        (void)p_wait;
    } else if (warp == 1) {
        // ---- MMA issue: the warp runs the loop (waits are warp-uniform), one elected lane issues
        if (n_ang > 0 && n_rounds > 0) {
            // B (MN-major, no swizzle, the TMA box [plane][row/8][chan][row%8]): LBO = 128 B between
            // 8-channel chunks, SBO = 256 B between 8-row groups, T_lo nb x 32 B after T_hi; slot
            // offsets are added to the 14-bit start-address field (addr >> 4).  A (TMEM): lane = voxel
            // row, column j = channels 2j, 2j+1 (8 columns per fp16 K = 16 tile; hi at +0, lo at +8)
            const uint64_t dT = umma_sdesc(smem_u32(ring), 128, 256);
            const uint32_t lo_off = (uint32_t)(a.nb * kK * 2) >> 4;
            int item = 0;
            long long p_wait = 0, p_free = 0, p_issue = 0;
            PROBE_T0(p_start);
            for (;; ++item) {
                const int s = item % kSi, sa = item % kAi;
                PROBE_T0(q1);
                tc_wait_mma(&afull[sa], (uint32_t)(item / kAi) & 1u);
                tc_wait_mma(&full[s], (uint32_t)(item / kSi) & 1u);
                PROBE_ADD(p_wait, q1);
                const uint32_t cnt = *reinterpret_cast<volatile uint32_t*>(&s_cnt[sa]);
                const int ns = (int)(cnt & 0xffu);
                tc_fence_after();
                for (int j = 0; j < ns; ++j) {
                    const uint32_t ctl = *reinterpret_cast<volatile uint32_t*>(&s_ctl[sa * kQ + j]);
                    const uint32_t acc = (ctl & kCtlAcc) ? 1u : 0u;
                    if (ctl & kCtlFree) {
                        PROBE_T0(q0);
                        tc_wait(&accfree[acc], (ctl & kCtlFreePh) ? 1u : 0u, 3, item);
                        tc_fence_after();
                        PROBE_ADD(p_free, q0);
                    }
                    PROBE_T0(q2);
                    if (elect_one()) {
                        const uint64_t th = dT + (uint64_t)((s * kSlot + j * kStep) >> 4), tl = th + lo_off;
                        const uint32_t ah = tmem + kAcol + kAslot * (uint32_t)sa + 16u * (uint32_t)j, al = ah + 8u;
                        const uint32_t td = tmem + acc * kNB;
                        const uint32_t idesc = kIdesc | (((ctl >> kCtlN) & 0xffu) << 1) << 17;  // (N/16)*2 = N>>3
#ifndef TF_TC_PROBE_NO_MMA  // probe builds only: timing without the MMAs
                        umma_f16_ts(td, ah, th, idesc, (ctl & kCtlFirst) ? 0u : 1u);
                        umma_f16_ts(td, al, th, idesc, 1u);
                        umma_f16_ts(td, ah, tl, idesc, 1u);
#else
                        (void)th, (void)tl, (void)ah, (void)al, (void)td, (void)idesc;
#endif
                        if (ctl & kCtlLast) umma_commit(&accfull[acc]);
                    }
                    __syncwarp();
                    PROBE_ADD(p_issue, q2);
                }
                if (elect_one()) umma_commit(&done[item % kB]);  // frees the item's tap and A slots
                __syncwarp();
                if (cnt & kCntEnd) break;
            }
            ++item;
#ifdef TF_TC_PROBE
            if (a.probe && lane == 0 && blockIdx.x < 1024) {
                a.probe[blockIdx.x * 16 + 2] = clock64() - p_start;
                a.probe[blockIdx.x * 16 + 3] = p_wait;
                a.probe[blockIdx.x * 16 + 4] = p_free;
                a.probe[blockIdx.x * 16 + 5] = p_issue;
                a.probe[blockIdx.x * 16 + 6] = item;
            }
#endif
            (void)p_wait, (void)p_free, (void)p_issue;
        }
    } else {
        // ---- weight groups: item i -> group i % kG; one voxel row per thread (TMEM lane quadrant =
        // warp % 4); column slice grp of the master sum
        const int grp = (warp - 2) >> 2;
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const bool real = m < kMV;  // rows kMV..127 of the MMA: zero weights, no output
        const int vx = m % kTX, vy = m / kTX;
        const float fdx = (float)vx, fdy = (float)vy;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);  // this warp's TMEM lanes
        int item_round = 0;  // items before this round (every role counts the same sequence)
        int blk_round = 0;   // accumulator blocks before this round (the ping-pong parity runs on)
        long long p_wait = 0, p_flush = 0;
        PROBE_T0(p_start);
        for (int r = 0; r < n_rounds; ++r) {
            const TcWork wk = tc_work(r * G + (int)blockIdx.x, a);
            const int slice = wk.n / kG;  // master columns of this thread's group (multiple of 4)
            // this thread's voxel (x, y) inside the requested tile?  Recomputed for the epilogue
            // rather than kept live through the angle loop (register pressure)
            auto voxel = [&](int& x, int& y) {
                x = (wk.tile % a.ntx) * kTX + vx;
                y = (wk.tile / a.ntx) * kTY + vy;
                return real && x < a.nx && y < a.ny && x >= a.x0 && x < a.x1 && y >= a.y0 && y < a.y1;
            };
            const double dX = (double)((wk.tile % a.ntx) * kTX) - a.cx, dY = (double)((wk.tile / a.ntx) * kTY) - a.cy;
            // this round's per-row scalings (the previous round's epilogue is done with them)
            named_bar_sync(1, 128 * kG);
            for (int i = threadIdx.x - 64; i < wk.n; i += 128 * kG) {
                const int e = wk.zr0 + i < a.n_rows ? a.e_rows[wk.zr0 + i] : 0;  // |e| <= 100: normal powers of two
                s_up[i] = __int_as_float((127 + e) << 23);
                s_dn[i] = __int_as_float((127 - e) << 23);
            }
            named_bar_sync(1, 128 * kG);
            float master[kNC];
#pragma unroll
            for (int j = 0; j < kNC; ++j) master[j] = 0.f;
            if (a.flags & TF_BP_ACCUMULATE) {  // continue unscaled partial sums: x 2^e is exact
                int x, y;
                if (voxel(x, y)) {
                    const int zc0 = wk.zr0 + grp * slice;
                    const float* src = a.vol + (size_t)y * a.nx + x;
#pragma unroll
                    for (int j = 0; j < kNC; ++j)
                        if (j < slice && zc0 + j < a.n_rows) master[j] = src[(size_t)(zc0 + j) * plane] * s_up[grp * slice + j];
                }
            }
            int flushed = 0;
            // master (+)= the accumulator of the round's next unflushed block, round to nearest, once its
            // MMAs retired; `block` waits for them, otherwise only a retired block is flushed
            auto flush = [&](bool block) {
                const int gb = blk_round + flushed, acc = gb & 1;
                const uint32_t ph = (uint32_t)(gb >> 1) & 1u;
                if (block) {
                    tc_wait(&accfull[acc], ph, 4, gb);
                } else if (!mbar_test(&accfull[acc], ph)) {  // test_wait: never parks the warp
                    return false;
                }
                tc_fence_after();
                // 8-column loads; a slice of 4 mod 8 reads 4 columns past it into master entries the
                // epilogue never writes
#pragma unroll
                for (int c = 0; c < kNC; c += 8) {
                    if (c < slice) {
                        uint32_t v[8];
#ifndef TF_TC_PROBE_NO_FLUSH  // probe builds only: timing without the TMEM reads
                        TC_LD8(tl + (uint32_t)(acc * kNB + grp * slice + c), v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#else
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] = 0u;
#endif
#pragma unroll
                        for (int j = 0; j < 8; ++j) master[c + j] = __fadd_rn(master[c + j], __uint_as_float(v[j]));
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&accfree[acc]);
                ++flushed;
                return true;
            };
            const bool last_round = r == n_rounds - 1;
            const uint32_t nctl = (uint32_t)(wk.n >> 4) << kCtlN;
            int st = 0;  // step of the round
            // this group's turn in item `item`: the A slot's previous item must retire (flush retired
            // blocks meanwhile); after its step's store, the warp's arrival
            auto slot_wait = [&](int item) {
                if (flushed < n_blk) flush(false);
                if (item >= kAi) {
                    const int x = item - kAi;
                    PROBE_T0(q4);
                    while (!tc_poll_w(&done[x % kB], (uint32_t)(x / kB) & 1u))
                        if (flushed < n_blk) flush(false);
                    PROBE_ADD(p_wait, q4);
                }
            };
            auto arrive = [&](int sa) {
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[sa]);
            };
            for (int g0 = 0; g0 < n_ang; g0 += 32) {
                const TcBatch bt = tc_batch(g0, n_ang, dX, dY, a);
                for (int i = 0; i < bt.n; ++i) {
                    const int nk = 1 + ((bt.two >> i) & 1);
                    // step j of every item is group j's: does angle i have one?
                    if (((st - grp) & (kQ - 1)) != 0 && (nk == 1 || ((st + 1 - grp) & (kQ - 1)) != 0)) {
                        st += nk;
                        continue;
                    }
                    const int ab = a.a0 + g0 + i;
                    const TcWin w = tc_bcast(bt.w, i);
                    const float t = fmaxf(fmaf(fdy, w.C, fmaf(fdx, w.B, w.F0)), 0.f);
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
                    for (int ks = 0; ks < nk; ++ks, ++st) {
                        const int j = st % kQ;
                        if (j != grp) continue;
                        const int item = item_round + st / kQ, sa = item % kAi;
                        slot_wait(item);
                        // tap o = floor(t) - 16 ks of this step's window; the pair (2u, 2u + 1) of
                        // halves holding it is jo = o >> 1 (o = -1: only f lands, in pair 0)
                        const int jo = real ? (o0 - kK * ks) >> 1 : -8;
                        uint32_t v[16];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            v[u] = u == jo ? Xh : (u == jo + 1 ? Yh : 0u);
                            v[8 + u] = u == jo ? Xl : (u == jo + 1 ? Yl : 0u);
                        }
                        tc_fence_after();
#ifndef TF_TC_PROBE_NO_WST  // probe builds only: timing without the TMEM weight stores
                        TC_ST16(tl + kAcol + kAslot * (uint32_t)sa + 16u * (uint32_t)j, v);
#else
                        if (v[0] == 0x12345678u && v[15] == 0x12345678u) TC_ST16(tl + kAcol + kAslot * (uint32_t)sa, v);
#endif
                        const bool round_end = g0 + i == n_ang - 1 && ks == nk - 1;
                        if (q == 0 && lane == 0) {
                            // the MMA warp's control word: accumulate = 0 (block's first step), commit the
                            // block (its last), accumulator, wait for the accumulator's flush (from the
                            // third block on) and that wait's phase, N / 16; the item's last step also
                            // writes the item's step count and the end of the CTA's work
                            const int g = ab - a.a0, gb = blk_round + ab / kP - blk0;
                            const bool first = ks == 0 && (g == 0 || ab % kP == 0);
                            const bool last = ks == nk - 1 && (g == n_ang - 1 || (ab + 1) % kP == 0);
                            s_ctl[sa * kQ + j] = (first ? kCtlFirst : 0u) | (last ? kCtlLast : 0u) |
                                                 ((gb & 1) ? kCtlAcc : 0u) | ((first && gb >= 2) ? kCtlFree : 0u) |
                                                 ((((gb >> 1) - 1) & 1) ? kCtlFreePh : 0u) | nctl;
                            if (j == kQ - 1 || round_end)
                                s_cnt[sa] = (uint32_t)(j + 1) | ((last_round && round_end) ? kCntEnd : 0u);
                        }
                        arrive(sa);
                    }
                }
            }
            // the round's last item may be short: the groups without a step in it still arrive
            if (st % kQ != 0 && grp >= st % kQ) {
                const int item = item_round + st / kQ;
                slot_wait(item);
                arrive(item % kAi);
            }
            PROBE_T0(q3);
            while (flushed < n_blk) flush(true);
            PROBE_ADD(p_flush, q3);
            item_round += (st + kQ - 1) / kQ;
            blk_round += n_blk;
            // ---- epilogue: master x 2^-e -> volume (fbp.py:247-251)
            int x, y;
            if (voxel(x, y)) {
                const int zc0 = wk.zr0 + grp * slice;  // first volume row of this thread's master columns
                const bool fin = (a.flags & TF_BP_FINALIZE) != 0;
                const bool zero = fin && tc_outside_fov(x, y, a);
                float* out = a.vol + (size_t)y * a.nx + x;
#pragma unroll
                for (int j = 0; j < kNC; ++j) {
                    const int zz = zc0 + j;
                    if (j < slice && zz < a.n_rows) {
                        float val = master[j] * s_dn[grp * slice + j];
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
                if (!last_round) {
                    const unsigned target = (unsigned)(r + 1) * (unsigned)G;
                    const long long t0 = clock64();
                    while (*reinterpret_cast<volatile unsigned*>(a.sync) < target) {
                        __nanosleep(64);
                        if (clock64() - t0 > 20000000000LL) __trap();
                    }
                    __threadfence();
                }
            }
        }
#ifdef TF_TC_PROBE
        if (a.probe && lane == 0 && blockIdx.x < 1024 && (warp == 2 || warp == 14)) {
            const int o = warp == 2 ? 7 : 10;
            a.probe[blockIdx.x * 16 + o] = clock64() - p_start;
            a.probe[blockIdx.x * 16 + o + 1] = p_wait;
            a.probe[blockIdx.x * 16 + o + 2] = p_flush;
        }
#endif
        (void)p_wait, (void)p_flush;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
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
        n += 1 + (tc_two_steps(tc_window(dX, dY, a.trig[a.a0 + g], a)) ? 1 : 0);
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

int launch_tc(const CUtensorMap& map, const TCArgs& a, cudaStream_t s) {
    auto* fn = bp_tc_kernel;
    TF_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    int dev = 0, sms = 0, per_sm = 0;
    TF_CUDA_TRY(cudaGetDevice(&dev));
    TF_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, kSmem));
    if (per_sm < 1) return set_error(TF_ERR_UNSUPPORTED, "bp_tc_kernel does not fit on an SM");
    // every CTA of a round must be resident for the lockstep barrier: a cooperative launch
    const unsigned grid = (unsigned)std::min<long long>((long long)sms * per_sm, a.n_work);
    TCArgs args = a;
    CUtensorMap m = map;
    void* kargs[] = {&m, &args};
    TF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kThreads), kargs, kSmem, s));
    return check_launch("bp_tc_kernel");
}

// z-blocks of a slab: as few as kNB allows, of equal height rounded up to 16 rows (the MMA's N
// granularity); the last block's N covers the remainder
struct TcBlocks {
    int nb, nzb, n_last;
};
TcBlocks tc_blocks(int n_rows) {
    TcBlocks b{};
    if (n_rows <= 0) return b;
    const int want = (n_rows + kNB - 1) / kNB;
    b.nb = std::min(kNB, ((n_rows + want - 1) / want + 15) / 16 * 16);
    b.nzb = (n_rows + b.nb - 1) / b.nb;
    b.n_last = (n_rows - (b.nzb - 1) * b.nb + 15) / 16 * 16;
    return b;
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
    const TcBlocks zb = tc_blocks(n_rows);

    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    CUtensorMap map;
    void* ws = const_cast<void*>(taps);
    void* data = tc_taps_ptr(p, ws, n_rows);
    // dim 0 = (channel, row-in-group) flattened: a box row is 16 channels x 8 rows = 256 contiguous
    // bytes; channel c starts at element 8 c.  dim 1 = 8-row group, dim 2 = (angle, plane).
    cuuint64_t dims[3] = {(cuuint64_t)8 * g.n_chan, (cuuint64_t)R8, (cuuint64_t)(2 * (taps_a1 - taps_a0))};
    cuuint64_t strides[2] = {(cuuint64_t)g.n_chan * 16u, (cuuint64_t)R8 * g.n_chan * 16u};
    cuuint32_t box[3] = {(cuuint32_t)(8 * kK), (cuuint32_t)(zb.nb / 8), 2u};  // T_hi and T_lo of one step
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
    a.nb = zb.nb;
    a.nzb = zb.nzb;
    a.n_last = zb.n_last;
    a.tx_bytes = 2 * zb.nb * kK * 2;
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
    a.n_work = a.n_tiles * zb.nzb;
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
    return launch_tc(map, a, s);
}

extern "C" int tf_bp_tc_work(const tf_bp_plan* p, int n_rows, int a0, int a1, int64_t* items,
                             int64_t* executed_updates, int64_t* mma_clocks) {
    if (!p || !items || !executed_updates || !mma_clocks) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    if (!(0 <= a0 && a0 <= a1 && a1 <= p->g.n_proj) || n_rows < 0)
        return set_error(TF_ERR_INVALID_ARGUMENT, "invalid rows/angles");
    const TcBlocks zb = tc_blocks(n_rows);
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
    *items = (int64_t)per_zblock * zb.nzb;
    *executed_updates = vox * (int64_t)n_rows * (a1 - a0);
    // 3 MMAs of 128 x N x 16 per item at N / 2 clk each, N the z-block's rows
    *mma_clocks = (int64_t)per_zblock * 3 * ((int64_t)(zb.nzb - 1) * zb.nb + zb.n_last) / 2;
    return TF_OK;
}

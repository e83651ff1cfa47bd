// K2: voxel-driven back-projection (replaces fbp.back_project, fbp.py:186-252).
//
// Data layout in HBM ("z-blocked staging", written by tf_bp_stage):
//   stage[(k * nzb + zb) * n_chan + c][zi]  fp32, zi in [0, 36)
// i.e. for every angle k and block of 32 detector rows zb, each channel c
// holds the 32 rows contiguously (+4 zero pad floats: a 144-B row pitch puts
// consecutive channels in distinct 16-B bank quads, so the LDS.128 gathers
// below are conflict-free without a swizzle).  Feather weights
// (fbp.py:242) are folded in while staging.
//
// Kernel structure (default variant: one CTA = 16x16 voxel columns x one
// 32-row z-block, 4 consumer warps + 1 producer warp, 3 CTAs per SM):
//   * the producer warp: per angle lane 0 computes, in fp64, the channel
//     window [c_lo, c_lo+W) the tile's rays hit and issues one
//     cp.async.bulk.tensor box {36, W, 1} into an 8-stage x 2-angle smem ring
//     (an mbarrier per slot, completed by the TMA transaction count).  It
//     refills a slot once every consumer has arrived on the slot's named
//     barrier (bar.sync parks the warp; no polling).  Out-of-detector
//     channels come back as zeros from the TMA OOB fill -- the reference's
//     zero guard.
//   * each consumer thread owns a pair of voxels along x x 32 rows (64
//     accumulators); per angle it forms t in fp32 *relative to the tile
//     origin* (origin and window offset in fp64: |error| ~1e-6 channels even
//     at 8192 channels, where a plain fp32 t would be off by ~5e-4), reads
//     the pair's 3 taps for all 32 rows with 3x8 LDS.128 (6 B of shared
//     memory per update) and accumulates with 96 packed FFMA2 using the
//     exact two-tap weights of each voxel (bit-identical to the 2-tap V1).
//   * epilogue: FoV mask evaluated in fp64 exactly as fbp.py:247-250, scale by
//     float32(angle_span / n_proj) (fbp.py:251), coalesced stores -- or, for
//     angle-split partials (RED), adds into each row's owner slab.
// Tiles wholly outside the field of view skip the angle loop.
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include <cuda_fp16.h>

#include "bp_plan.hpp"
#include "common.cuh"

namespace tf {
namespace {


// Consumer layouts.  A thread owns a VX x VY block of voxel columns and ZT of
// the tile's 32 rows; NT detector taps per block serve all its voxels:
//   V1 (1x1, NT=2, ZT=32): the classic two-tap gather, 8 B of smem per update;
//   pair (2x1, NT=3, ZT=32, the default): the pair's rays differ by
//       |cos|*scale <= 1 channel, so 3 taps serve both voxels, 6 B per update,
//       with each voxel's exact {1-f, f} weights (bit-identical to V1).
// Other blockings (2x2 / 4 taps, x-runs of 3, a 2x2 "role" kernel) were
// measured in round 1 (profiles/r01_bp_variants_*.jsonl) and
// lost to the pair kernel; they are no longer compiled into the library.
template <int VX, int VY, int NT, int ZT, int STAGES_, int APS_, bool PIPE_, int MINB_, int PW_>
struct Layout {
    static constexpr int TX = kTileShape[kShapeCuda][0], TY = kTileShape[kShapeCuda][1];  // voxel columns per CTA
    static constexpr int PW = PW_, PH = 8 / PW_;  // one 8-lane LDS.128 phase = PW x PH blocks
    static constexpr int STAGES = STAGES_, APS = APS_, RING = STAGES_ * APS_;  // smem ring of angle slots
    static constexpr bool PIPE = PIPE_;  // software-pipeline the next angle's setup under this angle's FMAs
    static constexpr int MINB = MINB_;
    static constexpr int VX_ = VX, VY_ = VY, NT_ = NT, ZT_ = ZT;
    static constexpr int BX = TX / VX, BY = TY / VY;   // blocks per tile
    static constexpr int COLS = BX * BY;               // threads per z-group
    static constexpr int ZG = kZB / ZT;                // z-groups
    static constexpr int NCT = COLS * ZG;              // consumer threads
    static constexpr int NCW = NCT / 32;               // consumer warps
    static constexpr int NTHREADS = NCT + 32;          // + TMA producer warp
    static constexpr int WX = BX / 8;                  // warps across a z-group (8x4 blocks each)
    static_assert(COLS % 32 == 0 && BX % 8 == 0 && BY % 4 == 0, "warp tiling");
    static_assert(NT == VX * VY + 1 || NT == 2, "V1 or the x-pair kernel");
};

struct BPArgs {
    const double2* trig;
    const int* order;  // blockIdx.x -> tile index (Morton order, FoV-active tiles first)
    float* vol;
    int a0, a1, nzb, n_rows, nx, ny, n_chan;
    int x0, x1, y0, y1;
    int ntx;
    int W, slot_bytes;
    int flags;
    double cx, cy, scale, axis, R2, sc2;
    float angle_wf;
    // TF_BP_REDUCE: row z's partial sums are added (red.global.add) into the
    // slab owning it, rdst[s] + (z - rrow0[s]) * plane (peer memory allowed)
    int a_base;  // first angle held in the staging buffer (0: it holds all n_proj)
    int n_rslabs;
    int rrow0[9];
    float* rdst[8];
};

__device__ __forceinline__ bool outside_fov(int x, int y, const BPArgs& a) {
    // ((x-cx)^2 + (y-cy)^2) * scale^2 > R^2, no FMA contraction (fbp.py:247-250)
    double dx = __dsub_rn((double)x, a.cx), dy = __dsub_rn((double)y, a.cy);
    double rr = __dmul_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), a.sc2);
    return rr > a.R2;
}

// acc[0..3] += t * w as two packed FFMA2 (sm_100 FP32x2; per lane the same
// fused, round-to-nearest operation as fmaf, so results are bit-identical)
// with w as the broadcast scalar operand: half the issue slots of 4 FFMA.
__device__ __forceinline__ void fma4(float2& a01, float2& a23, const float4& t, float w) {
    a01 = __ffma2_rn(make_float2(t.x, t.y), make_float2(w, w), a01);
    a23 = __ffma2_rn(make_float2(t.z, t.w), make_float2(w, w), a23);
}

template <class L, bool RED = false>  // RED: TF_BP_REDUCE epilogue (own instantiation: no register cost elsewhere)
__global__ void __launch_bounds__(L::NTHREADS, L::MINB)
    bp_kernel(const __grid_constant__ CUtensorMap map, const BPArgs args) {
    constexpr int VX = L::VX_, VY = L::VY_, NT = L::NT_, ZT = L::ZT_;
    constexpr int STAGES = L::STAGES, APS = L::APS;
    constexpr int TX = L::TX, TY = L::TY;
    extern __shared__ __align__(128) uint8_t smem[];
    // CTAs launch in blockIdx order and the resident set is a sliding window of
    // ~3 x 148 consecutive entries: a Morton order makes that window a compact
    // patch whose channel windows overlap, so the z-block's angle working set
    // stays in L2 instead of being re-read from HBM tile by tile.
    const int tile = args.order ? args.order[blockIdx.x] : (int)blockIdx.x;
    const int tx = tile % args.ntx, ty = tile / args.ntx, zb = blockIdx.y;
    const int X0 = tx * TX, Y0 = ty * TY;

    // ---- tile-level early outs (uniform over the CTA, before any barrier)
    const int xe = min(X0 + TX, args.nx), ye = min(Y0 + TY, args.ny);
    const int ux0 = max(X0, args.x0), ux1 = min(xe, args.x1);
    const int uy0 = max(Y0, args.y0), uy1 = min(ye, args.y1);
    if (ux0 >= ux1 || uy0 >= uy1) return;  // nothing of the requested tile here
    {
        // nearest voxel of the tile to the rotation centre decides "all outside"
        int nxv = (int)fmin(fmax(rint(args.cx), (double)X0), (double)(xe - 1));
        int nyv = (int)fmin(fmax(rint(args.cy), (double)Y0), (double)(ye - 1));
        bool all_out = true;
        for (int ddx = -1; ddx <= 1; ++ddx)
            for (int ddy = -1; ddy <= 1; ++ddy) {
                int xx = min(max(nxv + ddx, X0), xe - 1), yy = min(max(nyv + ddy, Y0), ye - 1);
                all_out = all_out && outside_fov(xx, yy, args);
            }
        if (all_out) {
            if (args.flags & TF_BP_FINALIZE) {
                const int nz = min(kZB, args.n_rows - zb * kZB);
                const size_t plane = (size_t)args.nx * args.ny;
                for (int i = threadIdx.x; i < TX * TY * nz; i += blockDim.x) {
                    int z = i / (TX * TY), r = i % (TX * TY);
                    int x = X0 + (r % TX), y = Y0 + (r / TX);
                    if (x >= ux0 && x < ux1 && y >= uy0 && y < uy1)
                        args.vol[(size_t)(zb * kZB + z) * plane + (size_t)y * args.nx + x] = 0.f;
                }
            }
            return;
        }
    }

    uint8_t* ring = smem;
    float4* prm = reinterpret_cast<float4*>(smem + STAGES * APS * args.slot_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(prm + STAGES * APS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();

    const int n_ang = args.a1 - args.a0;
    const int n_it = (n_ang + APS - 1) / APS;

    if (warp == L::NCW) {
        // ================= TMA producer (lane 0 issues; the warp waits)
        // A ring slot is refilled once every consumer thread has arrived on
        // the slot's named barrier: bar.sync parks the warp in hardware (a
        // polled mbarrier kept ~20% of the SM's issue slots busy spinning).
        if (lane == 0) tma_prefetch_desc(&map);
        const double dX = (double)X0 - args.cx, dY = (double)Y0 - args.cy;
        const uint32_t box_bytes = (uint32_t)(kZP * 4 * args.W);
        for (int it = 0; it < n_it; ++it) {
            const int s = it % STAGES;
            if (it >= STAGES) named_bar_sync(1 + s, L::NTHREADS);  // round it-STAGES consumed
            if (lane == 0) {
                const int kb = args.a0 + it * APS;
                const int na = min(APS, args.a1 - kb);
                int c_lo[APS];
                for (int a = 0; a < na; ++a) {
                    const double2 cs = args.trig[kb + a];
                    // t at the tile origin, same operation order as geometry.py:151-153
                    double t0 = __dadd_rn(__dmul_rn(dX, cs.x), __dmul_rn(dY, cs.y));
                    t0 = __dadd_rn(__dmul_rn(t0, args.scale), args.axis);
                    const double B = cs.x * args.scale, C = cs.y * args.scale;
                    const double tmin = t0 + fmin(0.0, B * (TX - 1)) + fmin(0.0, C * (TY - 1));
                    c_lo[a] = (int)floor(tmin);
                    prm[s * APS + a] = make_float4((float)(t0 - (double)c_lo[a]), (float)B, (float)C, 0.f);
                }
                mbar_arrive_expect_tx(&full[s], box_bytes * (uint32_t)na);
                for (int a = 0; a < na; ++a)
                    tma_load_3d(ring + (size_t)(s * APS + a) * args.slot_bytes, &map, &full[s], 0, c_lo[a],
                                (kb + a - args.a_base) * args.nzb + zb);
            }
            __syncwarp();
        }
        return;
    }

    // ================= consumers
    // z-group per warp (all lanes of a warp read the same 16-B column of a
    // tap row); a warp covers 8x4 blocks, each 8-lane LDS.128 phase a 4x2
    // patch, so a phase's tap rows stay within 8 consecutive channels ->
    // distinct bank quads (row pitch 144 B = 9 quads).
    const int zg = threadIdx.x / L::COLS;
    const int wg = (threadIdx.x % L::COLS) >> 5;
    const int q = lane >> 3, i8 = lane & 7;
    constexpr int QW = 8 / L::PW;  // phases across the warp's 8-block width
    const int bx = (wg % L::WX) * 8 + (q % QW) * L::PW + (i8 % L::PW);
    const int by = (wg / L::WX) * 4 + (q / QW) * L::PH + (i8 / L::PW);
    const int dx0 = bx * VX, dy0 = by * VY;
    const size_t plane = (size_t)args.nx * args.ny;
    const int zrow0 = zb * kZB + zg * ZT;                 // first volume row of this thread
    const int nz = min(ZT, args.n_rows - zrow0);          // may be <= 0 for a ragged last block

    float acc[VX * VY][ZT];
#pragma unroll
    for (int v = 0; v < VX * VY; ++v)
#pragma unroll
        for (int j = 0; j < ZT; ++j) acc[v][j] = 0.f;
    if (args.flags & TF_BP_ACCUMULATE) {
#pragma unroll
        for (int v = 0; v < VX * VY; ++v) {
            const int x = X0 + dx0 + (v % VX), y = Y0 + dy0 + (v / VX);
            if (x >= ux0 && x < ux1 && y >= uy0 && y < uy1) {
#pragma unroll
                for (int j = 0; j < ZT; ++j)
                    if (j < nz) acc[v][j] = args.vol[(size_t)(zrow0 + j) * plane + (size_t)y * args.nx + x];
            }
        }
    }

    // per-angle setup: detector coordinates -> tap row + interpolation weights
    const uint8_t* ring_z = ring + zg * ZT * 4;
    auto setup = [&](int g, const float*& p0, float (&w)[VX * VY][NT]) {
        const int slot = g % L::RING;  // RING need not be a power of 2
        const float4 p = prm[slot];
        const uint8_t* base = ring_z + slot * args.slot_bytes;
        if constexpr (NT == 2) {
            float t = fmaf((float)dy0, p.z, fmaf((float)dx0, p.y, p.x));
            t = fmaxf(t, 0.f);
            const float fl = floorf(t);
            const float f = t - fl;
            w[0][0] = 1.f - f;
            w[0][1] = f;
            p0 = reinterpret_cast<const float*>(base + (int)fl * kRowBytes);
        } else if constexpr (NT == 3) {
            // pair of voxels along x: their rays differ by |cos|*scale <= 1
            // channel, so taps fb..fb+2 cover both.  Weights are the exact
            // two-tap {1-f, f} of the 2-tap kernel, placed at o = floor(t)-fb.
            float t[VX * VY];
            float tmin = 3.0e38f;
#pragma unroll
            for (int v = 0; v < VX * VY; ++v) {
                t[v] = fmaxf(fmaf((float)(dy0 + v / VX), p.z, fmaf((float)(dx0 + v % VX), p.y, p.x)), 0.f);
                tmin = fminf(tmin, t[v]);
            }
            const float fb = floorf(tmin);
#pragma unroll
            for (int v = 0; v < VX * VY; ++v) {
                const float fl = floorf(t[v]);
                const float f = t[v] - fl;
                const float g0 = 1.f - f;
                const bool hi = fl > fb;  // o == 1
                w[v][0] = hi ? 0.f : g0;
                w[v][1] = hi ? g0 : f;
                w[v][2] = hi ? f : 0.f;
            }
            p0 = reinterpret_cast<const float*>(base + (int)fb * kRowBytes);
        }
    };
    auto accumulate = [&](const float* p0, const float (&w)[VX * VY][NT]) {
#pragma unroll
        for (int c = 0; c < ZT / 4; ++c) {
            float4 T[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) T[j] = *reinterpret_cast<const float4*>(p0 + j * kZP + 4 * c);
#pragma unroll
            for (int v = 0; v < VX * VY; ++v) {
                float2 a01 = make_float2(acc[v][4 * c + 0], acc[v][4 * c + 1]);
                float2 a23 = make_float2(acc[v][4 * c + 2], acc[v][4 * c + 3]);
#pragma unroll
                for (int j = 0; j < NT; ++j) fma4(a01, a23, T[j], w[v][j]);
                acc[v][4 * c + 0] = a01.x;
                acc[v][4 * c + 1] = a01.y;
                acc[v][4 * c + 2] = a23.x;
                acc[v][4 * c + 3] = a23.y;
            }
        }
    };
    auto wait_full = [&](int g) {  // first angle of a stage
        const int it = g / APS;
        mbar_wait(&full[it % STAGES], (uint32_t)(it / STAGES) & 1u);
    };
    auto release = [&](int g) {  // last angle of a stage (or of the launch)
        const int it = g / APS;
        if (it + STAGES < n_it) named_bar_arrive(1 + it % STAGES, L::NTHREADS);  // the producer refills it
    };

    if constexpr (!L::PIPE) {
        for (int g = 0; g < n_ang; ++g) {
            if (g % APS == 0) wait_full(g);
            const float* p0;
            float w[VX * VY][NT];
            setup(g, p0, w);
            accumulate(p0, w);
            if (g % APS == APS - 1 || g == n_ang - 1) release(g);
        }
    } else if (n_ang > 0) {
        wait_full(0);
        const float* p0;
        float w[VX * VY][NT];
        setup(0, p0, w);
        for (int g = 0; g < n_ang; ++g) {
            const int gn = g + 1;
            if (gn < n_ang && gn % APS == 0) wait_full(gn);
            const float* q0;
            float wn[VX * VY][NT];
            setup(min(gn, n_ang - 1), q0, wn);  // independent of this angle's FMAs
            accumulate(p0, w);
            if (gn % APS == 0 || gn == n_ang) release(g);
            p0 = q0;
#pragma unroll
            for (int v = 0; v < VX * VY; ++v)
#pragma unroll
                for (int j = 0; j < NT; ++j) w[v][j] = wn[v][j];
        }
    }

    if constexpr (RED) {
        // angle-split partials: fire-and-forget adds into each row's owner
        // (NVLink peer stores when the owner is another GPU); the reduction IS
        // this kernel's epilogue, overlapped with the other tiles' angle loops
#pragma unroll
        for (int j = 0; j < ZT; ++j) {
            if (j >= nz) break;
            const int z = zrow0 + j;
            float* base = nullptr;
#pragma unroll
            for (int s = 0; s < 8; ++s)  // constant indices: no local copy of the table
                if (s < args.n_rslabs && z >= args.rrow0[s] && z < args.rrow0[s + 1])
                    base = args.rdst[s] + (size_t)(z - args.rrow0[s]) * plane;
#pragma unroll
            for (int v = 0; v < VX * VY; ++v) {
                const int x = X0 + dx0 + (v % VX), y = Y0 + dy0 + (v / VX);
                if (x >= ux0 && x < ux1 && y >= uy0 && y < uy1) atomicAdd(base + (size_t)y * args.nx + x, acc[v][j]);
            }
        }
        return;
    }
#pragma unroll
    for (int v = 0; v < VX * VY; ++v) {
        const int x = X0 + dx0 + (v % VX), y = Y0 + dy0 + (v / VX);
        if (!(x >= ux0 && x < ux1 && y >= uy0 && y < uy1)) continue;
        float scale = 1.f;
        bool zero = false;
        if (args.flags & TF_BP_FINALIZE) {
            scale = args.angle_wf;
            zero = outside_fov(x, y, args);
        }
        float* out = args.vol + (size_t)zrow0 * plane + (size_t)y * args.nx + x;
#pragma unroll
        for (int j = 0; j < ZT; ++j)
            if (j < nz) out[(size_t)j * plane] = zero ? 0.f : acc[v][j] * scale;
    }
}

// ---- staging: angle-major rows -> z-blocked, feather-weighted ------------
// One block turn = 32 rows x 64 channels of one (angle, z-block): float4
// loads along channels (coalesced rows), transposed through shared memory,
// written back as 64 contiguous 144-B channel rows (fully coalesced float4
// stores, pad floats zeroed).
__global__ void __launch_bounds__(256) stage_kernel(const float* __restrict__ sino, float* __restrict__ stage,
                                                    const float* __restrict__ w, int n_proj, int n_chan,
                                                    int rows_per_angle, int r0, int n_rows, int nzb) {
    constexpr int CB = 64;                    // channels per turn
    __shared__ float tile[kZB][CB + 1];       // +1: conflict-light column reads
    const int nch = (n_chan + CB - 1) / CB;
    const long long total = (long long)n_proj * nzb * nch;
    const bool vec = (n_chan % 4) == 0 && (reinterpret_cast<uintptr_t>(sino) & 15) == 0;  // float4-aligned rows
    for (long long blk = blockIdx.x; blk < total; blk += gridDim.x) {
        const int cb = (int)(blk % nch);
        const long long kz = blk / nch;
        const int zb = (int)(kz % nzb);
        const int k = (int)(kz / nzb);
        const int c0 = cb * CB;
        // load 32 rows x 64 channels: 512 float4, 2 per thread, both in flight
        float4 v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int i = threadIdx.x + u * 256;
            const int zi = i >> 4, c = (i & 15) * 4;
            const int row = zb * kZB + zi;
            const size_t off = ((size_t)k * rows_per_angle + r0 + row) * n_chan + c0 + c;
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < n_rows) {
                if (vec && c0 + c + 3 < n_chan) {
                    v[u] = __ldcs(reinterpret_cast<const float4*>(sino + off));
                } else {
                    if (c0 + c + 0 < n_chan) v[u].x = sino[off + 0];
                    if (c0 + c + 1 < n_chan) v[u].y = sino[off + 1];
                    if (c0 + c + 2 < n_chan) v[u].z = sino[off + 2];
                    if (c0 + c + 3 < n_chan) v[u].w = sino[off + 3];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int i = threadIdx.x + u * 256;
            const int zi = i >> 4, c = (i & 15) * 4;
            // feather after the filter (fbp.py:242), fp32 product
            tile[zi][c + 0] = v[u].x * (c0 + c + 0 < n_chan ? w[c0 + c + 0] : 0.f);
            tile[zi][c + 1] = v[u].y * (c0 + c + 1 < n_chan ? w[c0 + c + 1] : 0.f);
            tile[zi][c + 2] = v[u].z * (c0 + c + 2 < n_chan ? w[c0 + c + 2] : 0.f);
            tile[zi][c + 3] = v[u].w * (c0 + c + 3 < n_chan ? w[c0 + c + 3] : 0.f);
        }
        __syncthreads();
        // write 64 channels x 36 floats = 576 contiguous float4
        float* dst = stage + (((size_t)k * nzb + zb) * n_chan + c0) * kZP;
        const int nc = min(CB, n_chan - c0);
        for (int i = threadIdx.x; i < nc * (kZP / 4); i += 256) {
            const int c = i / (kZP / 4), z4 = (i % (kZP / 4)) * 4;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            if (z4 < kZB) o = make_float4(tile[z4][c], tile[z4 + 1][c], tile[z4 + 2][c], tile[z4 + 3][c]);
            *reinterpret_cast<float4*>(dst + (size_t)c * kZP + z4) = o;
        }
        __syncthreads();
    }
}

template <class L>
int bp_smem_bytes(int slot_bytes) {
    return L::RING * slot_bytes + L::RING * (int)sizeof(float4) + 2 * L::STAGES * (int)sizeof(uint64_t);
}

}  // namespace

PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_encodeTiled_t>(p);
        return (PFN_encodeTiled_t) nullptr;
    }();
    return fn;
}
}  // namespace tf

namespace tf {
namespace {
// kernel configurations (VX, VY, taps, rows/thread, stages, angles/stage, pipelined setup, min CTAs/SM, phase width)
using V1Cfg = Layout<1, 1, 2, 32, 4, 4, false, 2, 4>;
using PairCfg = Layout<2, 1, 3, 32, 8, 2, true, 3, 2>;

bool tile_order_enabled() {
    static int v = [] {
        const char* e = getenv("TF_BP_MORTON");  // benchmarking knob: 0 = row-major tile launch order
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

// the x-pair kernel needs |cos| * scale <= 1 (3 taps per pair); V1 otherwise or on request
bool use_v1(const tf_bp_plan* p, int flags) { return (flags & TF_BP_KERNEL_V1) || p->scale > 1.0; }

// smem bytes gathered per update: 16 B per LDS.128 of 4 rows x taps / voxels
double bytes_per_update(bool v1) { return v1 ? 8.0 : 6.0; }

template <class L, bool RED = false>
int launch_bp(const CUtensorMap& map, const BPArgs& a, dim3 grid, void* stream) {
    const int smem = bp_smem_bytes<L>(a.slot_bytes);
    TF_CUDA_TRY(cudaFuncSetAttribute(bp_kernel<L, RED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    bp_kernel<L, RED><<<grid, L::NTHREADS, smem, as_stream(stream)>>>(map, a);
    return TF_OK;
}
}  // namespace
}  // namespace tf

using namespace tf;

namespace tf {
const float* bp_plan_weights(const tf_bp_plan* p) { return p->g.scan_mode ? p->d_w : nullptr; }
int bp_plan_n_chan(const tf_bp_plan* p) { return p->g.n_chan; }
}  // namespace tf

extern "C" int tf_offset_weights(const tf_geometry* g, int band, double* w) {
    if (!g || !w) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    const int n = g->n_chan;
    if (g->scan_mode == 0) {  // fbp.py:157-158
        for (int i = 0; i < n; ++i) w[i] = 1.0;
        return TF_OK;
    }
    if (band < 1) return set_error(TF_ERR_INVALID_ARGUMENT, "feather band must be >= 1 channel");
    const double c0 = (n - 1) / 2.0 - g->offset_chan;  // axis_channel, geometry.py:64-67
    for (int i = 0; i < n; ++i) {                      // fbp.py:161-183
        const double c = (double)i;
        const double near_edge = g->offset_chan > 0 ? c : (double)(n - 1) - c;
        const double own = std::min(std::max(near_edge / band, 0.0), 1.0);
        const double m = 2.0 * c0 - c;
        double other = 0.0;
        if (m >= 0 && m <= n - 1) {
            const double mn = g->offset_chan > 0 ? m : (double)(n - 1) - m;
            other = std::min(std::max(mn / band, 0.0), 1.0);
        }
        const double tot = own + other;
        w[i] = tot > 0 ? own / tot : 0.0;
    }
    return TF_OK;
}

extern "C" int tf_bp_plan_create(const tf_geometry* g, int feather_band, tf_bp_plan** plan) {
    if (!g || !plan) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    *plan = nullptr;
    if (g->n_proj < 1 || g->n_rows < 1 || g->n_chan < 2 || g->nx < 2 || g->ny < 2)
        return set_error(TF_ERR_INVALID_ARGUMENT, "invalid geometry sizes");
    if (!(g->angle_span > 0) || !(g->pixel_pitch > 0) || !(g->voxel_pitch > 0))
        return set_error(TF_ERR_INVALID_ARGUMENT, "spans and pitches must be positive");
    if (g->scan_mode == 0 && g->offset_chan != 0)
        return set_error(TF_ERR_INVALID_ARGUMENT, "normal scan requires offset_chan == 0");
    std::vector<double> w(g->n_chan);
    int st = tf_offset_weights(g, feather_band, w.data());
    if (st) return st;
    auto* p = new tf_bp_plan();
    p->g = *g;
    p->feather_band = feather_band;
    p->scale = g->voxel_pitch / g->pixel_pitch;
    // window: max over angles of a 16x16 tile's channel extent + taps + floor slack
    const double ext = std::sqrt(15.0 * 15.0 * 2) * p->scale;
    if (bp_smem_bytes<V1Cfg>((kRowBytes * (int)std::ceil(ext + 3.0) + 127) / 128 * 128) > 227 * 1024) {
        delete p;
        return set_error(TF_ERR_UNSUPPORTED, "voxel/pixel pitch ratio %.3g too large for the tile window",
                         p->scale);
    }
    p->cx = (g->nx - 1) / 2.0;
    p->cy = (g->ny - 1) / 2.0;
    p->axis = (g->n_chan - 1) / 2.0 - g->offset_chan;
    const double half = (g->n_chan - 1) / 2.0;  // fbp.py:134-144
    const double R = g->scan_mode ? half + std::fabs((double)g->offset_chan) : half;
    p->R2 = R * R;
    p->sc2 = p->scale * p->scale;
    const double step = g->angle_span / g->n_proj;
    p->angle_wf = (float)step;
    // tile launch order per tile shape: FoV-active tiles (same fp64 test as
    // the kernel's early-out) in Morton order, then the inactive ones
    std::vector<int> orders[kNumTileShapes];
    for (int shape = 0; shape < kNumTileShapes; ++shape) {
        const int TXs = kTileShape[shape][0], TYs = kTileShape[shape][1];
        const int ntx = (g->nx + TXs - 1) / TXs, nty = (g->ny + TYs - 1) / TYs;
        std::vector<int> act, inact;
        for (int t = 0; t < ntx * nty; ++t) {
            const int X0 = (t % ntx) * TXs, Y0 = (t / ntx) * TYs;
            const int xe = std::min(X0 + TXs, g->nx), ye = std::min(Y0 + TYs, g->ny);
            const int nxv = (int)std::min(std::max(std::nearbyint(p->cx), (double)X0), (double)(xe - 1));
            const int nyv = (int)std::min(std::max(std::nearbyint(p->cy), (double)Y0), (double)(ye - 1));
            bool all_out = true;
            for (int ddx = -1; ddx <= 1; ++ddx)
                for (int ddy = -1; ddy <= 1; ++ddy) {
                    const int xx = std::min(std::max(nxv + ddx, X0), xe - 1), yy = std::min(std::max(nyv + ddy, Y0), ye - 1);
                    volatile double dx = (double)xx - p->cx, dy = (double)yy - p->cy;
                    volatile double s2 = dx * dx;
                    volatile double t2 = dy * dy;
                    volatile double rr = (s2 + t2) * p->sc2;
                    all_out = all_out && (rr > p->R2);
                }
            (all_out ? inact : act).push_back(t);
        }
        auto morton = [&](int t) {
            unsigned x = (unsigned)(t % ntx), y = (unsigned)(t / ntx), m = 0;
            for (int b = 0; b < 16; ++b) m |= ((x >> b) & 1u) << (2 * b) | ((y >> b) & 1u) << (2 * b + 1);
            return m;
        };
        std::stable_sort(act.begin(), act.end(), [&](int a, int b) { return morton(a) < morton(b); });
        p->n_active[shape] = (int)act.size();
        p->n_tiles[shape] = ntx * nty;
        act.insert(act.end(), inact.begin(), inact.end());
        orders[shape] = act;
    }
    std::vector<double2> trig(g->n_proj);
    for (int k = 0; k < g->n_proj; ++k) {  // theta_k = k * (span / n_proj), geometry.py:69-70
        const double th = (double)k * step;
        trig[k] = make_double2(cos(th), sin(th));
    }
    std::vector<float> wf(g->n_chan);
    for (int i = 0; i < g->n_chan; ++i) wf[i] = (float)w[i];
    cudaError_t e = cudaMalloc(&p->d_trig, sizeof(double2) * g->n_proj);
    for (int s = 0; s < kNumTileShapes && e == cudaSuccess; ++s) {
        p->h_order[s] = new int[orders[s].size()];
        std::copy(orders[s].begin(), orders[s].end(), p->h_order[s]);
        e = cudaMalloc(&p->d_order[s], sizeof(int) * orders[s].size());
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_order[s], orders[s].data(), sizeof(int) * orders[s].size(), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMalloc(&p->d_w, sizeof(float) * g->n_chan);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_trig, trig.data(), sizeof(double2) * g->n_proj, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_w, wf.data(), sizeof(float) * g->n_chan, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        tf_bp_plan_destroy(p);
        return set_error(TF_ERR_CUDA, "bp plan setup failed: %s", cudaGetErrorString(e));
    }
    *plan = p;
    return TF_OK;
}

extern "C" int tf_bp_plan_destroy(tf_bp_plan* p) {
    if (!p) return TF_OK;
    cudaFree(p->d_trig);
    cudaFree(p->d_w);
    for (int s = 0; s < kNumTileShapes; ++s) {
        cudaFree(p->d_order[s]);
        delete[] p->h_order[s];
    }
    delete p;
    return TF_OK;
}

extern "C" int64_t tf_bp_stage_bytes(const tf_bp_plan* p, int n_rows) {
    if (!p || n_rows < 0) return -1;
    const int64_t nzb = (n_rows + kZB - 1) / kZB;
    return (int64_t)p->g.n_proj * nzb * p->g.n_chan * kZP * (int64_t)sizeof(float);
}

extern "C" int tf_bp_stage(const tf_bp_plan* p, const float* sino, int rows_per_angle, int r0, int r1,
                           void* stage, void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null bp plan");
    if (!(0 <= r0 && r0 <= r1 && r1 <= rows_per_angle))
        return set_error(TF_ERR_INVALID_ARGUMENT, "row range (%d, %d) out of bounds", r0, r1);
    const int n_rows = r1 - r0;
    if (n_rows == 0) return TF_OK;
    if (!sino || !stage) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    const int nzb = (n_rows + kZB - 1) / kZB;
    const long long total = (long long)p->g.n_proj * nzb * ((p->g.n_chan + 63) / 64);
    const int grid = (int)std::min<long long>(total, 148LL * 16);
    stage_kernel<<<grid, 256, 0, as_stream(stream)>>>(sino, static_cast<float*>(stage), p->d_w, p->g.n_proj,
                                                      p->g.n_chan, rows_per_angle, r0, n_rows, nzb);
    return check_launch("stage_kernel");
}

namespace tf {
namespace {
struct ReduceMap {
    int n;
    int row0[9];
    float* dst[8];
};

int backproject_impl(const tf_bp_plan* p, const void* stage, int n_rows, float* vol, int a0, int a1, int x0,
                     int x1, int y0, int y1, int flags, void* stream, const ReduceMap* rm, int a_base = 0) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null bp plan");
    const tf_geometry& g = p->g;
    if (!(0 <= a0 && a0 <= a1 && a1 <= g.n_proj))
        return set_error(TF_ERR_INVALID_ARGUMENT, "angle range (%d, %d) out of bounds", a0, a1);
    if (!(0 <= x0 && x0 <= x1 && x1 <= g.nx && 0 <= y0 && y0 <= y1 && y1 <= g.ny))
        return set_error(TF_ERR_INVALID_ARGUMENT, "tile (%d, %d, %d, %d) out of bounds", x0, x1, y0, y1);
    if (n_rows < 0) return set_error(TF_ERR_INVALID_ARGUMENT, "n_rows must be >= 0");
    if (n_rows == 0 || x0 == x1 || y0 == y1) return TF_OK;
    if (!stage || (!vol && !rm)) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    const int nzb = (n_rows + kZB - 1) / kZB;
    if (a0 == a1 && !(flags & TF_BP_FINALIZE)) return TF_OK;

    // kernel: the x-pair gather needs the pair's rays within one channel
    // (|cos| * voxel/pixel pitch ratio <= 1); else the 2-tap V1
    const bool v1 = use_v1(p, flags);
    const int shape = kShapeCuda;
    const int TXv = kTileShape[shape][0], TYv = kTileShape[shape][1];
    const double ext = std::sqrt((double)(TXv - 1) * (TXv - 1) + (double)(TYv - 1) * (TYv - 1)) * p->scale;
    const int W = (int)std::ceil(ext + (v1 ? 3.0 : 4.0));

    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    CUtensorMap map;
    cuuint64_t dims[3] = {(cuuint64_t)kZP, (cuuint64_t)g.n_chan, (cuuint64_t)(g.n_proj - a_base) * (cuuint64_t)nzb};
    cuuint64_t strides[2] = {(cuuint64_t)kRowBytes, (cuuint64_t)kRowBytes * (cuuint64_t)g.n_chan};
    cuuint32_t box[3] = {(cuuint32_t)kZP, (cuuint32_t)W, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(stage), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_error(TF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);

    BPArgs a{};
    a.trig = p->d_trig;
    a.order = tile_order_enabled() ? p->d_order[shape] : nullptr;
    a.vol = vol;
    a.a0 = a0;
    a.a1 = a1;
    a.nzb = nzb;
    a.n_rows = n_rows;
    a.nx = g.nx;
    a.ny = g.ny;
    a.n_chan = g.n_chan;
    a.x0 = x0;
    a.x1 = x1;
    a.y0 = y0;
    a.y1 = y1;
    a.ntx = (g.nx + TXv - 1) / TXv;
    a.W = W;
    a.slot_bytes = ((kRowBytes * W) + 127) / 128 * 128;
    a.flags = flags;
    a.cx = p->cx;
    a.cy = p->cy;
    a.scale = p->scale;
    a.axis = p->axis;
    a.R2 = p->R2;
    a.sc2 = p->sc2;
    a.angle_wf = p->angle_wf;
    a.a_base = a_base;
    if (rm) {
        a.n_rslabs = rm->n;
        for (int s = 0; s <= rm->n; ++s) a.rrow0[s] = rm->row0[s];
        for (int s = 0; s < rm->n; ++s) a.rdst[s] = rm->dst[s];
    }
    const int nty = (g.ny + TYv - 1) / TYv;
    dim3 grid((unsigned)(a.ntx * nty), (unsigned)nzb);
    int st;
    if (flags & TF_BP_REDUCE)  // reduce epilogue (own instantiations)
        st = v1 ? launch_bp<V1Cfg, true>(map, a, grid, stream) : launch_bp<PairCfg, true>(map, a, grid, stream);
    else
        st = v1 ? launch_bp<V1Cfg>(map, a, grid, stream) : launch_bp<PairCfg>(map, a, grid, stream);
    if (st) return st;
    return check_launch("bp_kernel");
}
}  // namespace
}  // namespace tf

extern "C" int tf_backproject(const tf_bp_plan* p, const void* stage, int n_rows, float* vol, int a0, int a1,
                              int x0, int x1, int y0, int y1, int flags, void* stream) {
    return backproject_impl(p, stage, n_rows, vol, a0, a1, x0, x1, y0, y1, flags & ~TF_BP_REDUCE, stream, nullptr);
}

extern "C" int tf_bp_kernel_info(const tf_bp_plan* p, int flags, int n_rows, int a0, int a1, double* bytes,
                                 int64_t* executed_updates) {
    if (!p || !bytes || !executed_updates) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    *bytes = bytes_per_update(use_v1(p, flags));
    const int shape = kShapeCuda;
    const int64_t tile_vox = kTileShape[shape][0] * kTileShape[shape][1];
    const int64_t rows = (int64_t)((n_rows + kZB - 1) / kZB) * kZB;
    *executed_updates = (int64_t)p->n_active[shape] * tile_vox * rows * (int64_t)(a1 - a0);
    return TF_OK;
}

extern "C" int tf_bp_smem_bytes_per_update(const tf_bp_plan* p, int flags, double* bytes) {
    if (!p || !bytes) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    *bytes = bytes_per_update(use_v1(p, flags));
    return TF_OK;
}

namespace tf {
namespace {
// FoV mask + angle weight of fbp.py:247-251 on unscaled partial sums (the
// TF_BP_FINALIZE epilogue as a separate pass, for reduced angle-split sums)
__global__ void finalize_kernel(float* __restrict__ vol, long long n, int nx, int ny, double cx, double cy,
                                double sc2, double R2, float wf) {
    const long long plane = (long long)nx * ny;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i % plane;
        const int x = (int)(r % nx), y = (int)(r / nx);
        const double dx = __dsub_rn((double)x, cx), dy = __dsub_rn((double)y, cy);
        const double rr = __dmul_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), sc2);
        vol[i] = rr > R2 ? 0.f : vol[i] * wf;
    }
}
}  // namespace
}  // namespace tf

extern "C" int tf_bp_finalize(const tf_bp_plan* p, float* vol, int n_rows, void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null bp plan");
    if (n_rows < 0) return set_error(TF_ERR_INVALID_ARGUMENT, "n_rows must be >= 0");
    if (n_rows == 0) return TF_OK;
    if (!vol) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    const long long n = (long long)n_rows * p->g.nx * p->g.ny;
    const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    finalize_kernel<<<grid, 256, 0, as_stream(stream)>>>(vol, n, p->g.nx, p->g.ny, p->cx, p->cy, p->sc2, p->R2,
                                                          p->angle_wf);
    return check_launch("finalize_kernel");
}

extern "C" int tf_backproject_reduce(const tf_bp_plan* p, const void* stage, int n_rows, int a0, int a1, int n_slabs,
                                     const int32_t* slab_row0, void* const* slab_dst, int flags, void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null bp plan");
    if (n_slabs < 1 || n_slabs > 8 || !slab_row0 || !slab_dst)
        return set_error(TF_ERR_INVALID_ARGUMENT, "invalid slab map");
    if (slab_row0[0] != 0 || slab_row0[n_slabs] != n_rows)
        return set_error(TF_ERR_INVALID_ARGUMENT, "slab rows must cover [0, n_rows)");
    for (int s = 0; s < n_slabs; ++s) {
        if (slab_row0[s + 1] < slab_row0[s]) return set_error(TF_ERR_INVALID_ARGUMENT, "slab rows must ascend");
        if (!slab_dst[s] && slab_row0[s + 1] > slab_row0[s])
            return set_error(TF_ERR_INVALID_ARGUMENT, "null slab destination");
    }
    ReduceMap rm;
    rm.n = n_slabs;
    for (int s = 0; s <= n_slabs; ++s) rm.row0[s] = slab_row0[s];
    for (int s = 0; s < n_slabs; ++s) rm.dst[s] = static_cast<float*>(slab_dst[s]);
    return backproject_impl(p, stage, n_rows, nullptr, a0, a1, 0, p->g.nx, 0, p->g.ny,
                            (flags & TF_BP_KERNEL_V1) | TF_BP_REDUCE, stream, &rm, a0);
}

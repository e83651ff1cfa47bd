// K2-TC's MMA ring in isolation, on every SM: per item 3 tcgen05.mma
// kind::f16 (M = 128, N = 256, K = 16; A K-major, B MN-major, SWIZZLE_NONE,
// the kernel's shared-memory layouts) into one TMEM accumulator and one
// tcgen05.commit onto the slot's "empty" mbarrier; a producer warp waits
// "empty" and arrives on "full" (no data), the MMA warp waits "full".
//   -DNOWAIT     : no ring (MMAs + commits back to back)
//   -DPROBE_A    : A in the layout of tools/micro/umma_probe.cu (LBO = 2 KB, SBO = 128 B)
//   -DPAIR       : the MMA warp waits two slots and issues 6 MMAs + 2 commits per round
//   -DBLOCKS     : two accumulators alternating every 16 items (accumulate = 0 at a block's first
//                  item, a commit on an "accfull" barrier at its last), as the kernel's RN blocks
//   -DBATCH      : every 32 items the MMA warp loads 32 (cos, sin) pairs and does the kernel's fp64
//                  window arithmetic + a ballot (tc_batch)
//   -DGROUPS     : + 16 "weight" warps in 4 groups of 4 (group g: items g mod 4), each warp waits
//                  "empty" and arrives on "full" (count 1 + 4), as the kernel's weight producers
// Prints clk per item (mean over 148 CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ring_probe ring_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mma(uint32_t td, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                 ::"r"(td), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(p));
    return p != 0;
}

constexpr int kS = 8, NR = 256, TAP = NR * 16 * 2, WP = 128 * 16 * 2, SLOT = 2 * TAP + 2 * WP;

#ifdef GROUPS
constexpr int kThr = 64 + 512;
#else
constexpr int kThr = 64;
#endif
__global__ void __launch_bounds__(kThr, 1) ring(int items, long long* out, const double2* trig) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kS * SLOT);
    uint64_t* empty = full + kS;
    uint64_t* accfull = empty + kS;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(accfull + 2);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kS * SLOT / 4; i += kThr) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // 1.0h
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
#ifdef GROUPS
        for (int s = 0; s < kS; ++s) { mbar_init(&full[s], 5); mbar_init(&empty[s], 1); }
#else
        for (int s = 0; s < kS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
#endif
        mbar_init(&accfull[0], 1);
        mbar_init(&accfull[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    if (warp == 0) {  // producer: no data, just the ring
#ifndef NOWAIT
        for (int it = 0; it < items; ++it) {
            const int s = it % kS;
            if (it >= kS) mbar_wait(&empty[s], ((it / kS) - 1) & 1);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&full[s]);
        }
#endif
    } else if (warp >= 2) {
#ifdef GROUPS
        const int grp = (warp - 2) >> 2;
        for (int it = grp; it < items; it += 4) {
            const int s = it % kS;
            if (it >= kS) mbar_wait(&empty[s], ((it / kS) - 1) & 1);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&full[s]);
        }
#endif
    } else {
        constexpr uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(NR >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t dT = sdesc(su32(smem), 128, 256);
#ifdef PROBE_A
        const uint64_t dW = sdesc(su32(smem + 2 * TAP), 2048, 128);
#else
        const uint64_t dW = sdesc(su32(smem + 2 * TAP), 128, 256);
#endif
        long long t0 = clock64();
#ifdef PAIR
        for (int it = 0; it < items; it += 2) {
            const int s = it % kS;
#ifndef NOWAIT
            mbar_wait(&full[s], (it / kS) & 1);
            mbar_wait(&full[s + 1], (it / kS) & 1);
#endif
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (elect_one()) {
                for (int u = 0; u < 2; ++u) {
                    const uint64_t so = (uint64_t)(((s + u) * SLOT) >> 4);
                    const uint64_t th = dT + so, tl = th + (TAP >> 4), wh = dW + so, wl = wh + (WP >> 4);
                    mma(tmem, wh, th, idesc, (it + u) ? 1u : 0u);
                    mma(tmem, wl, th, idesc, 1u);
                    mma(tmem, wh, tl, idesc, 1u);
                    commit(&empty[s + u]);
                }
            }
            __syncwarp();
        }
#else
        double acc_b = 0.0;
        for (int it = 0; it < items; ++it) {
            const int s = it % kS;
#ifdef BATCH
            if (it % 32 == 0) {
                const int lane = threadIdx.x & 31;
                const double2 cs = trig[(it + lane) % 1024];
                double t0 = __dadd_rn(__dmul_rn(3.0, cs.x), __dmul_rn(5.0, cs.y));
                t0 = __dadd_rn(__dmul_rn(t0, 1.0), 1023.5);
                const double tmin = t0 + fmin(0.0, cs.x * 10) + fmin(0.0, cs.y * 10);
                const int c = (int)floor(tmin);
                const unsigned two = __ballot_sync(0xffffffffu, (float)(t0 - c) > 14.9f);
                acc_b += (double)two + c;
            }
#endif
#ifndef NOWAIT
            mbar_wait(&full[s], (it / kS) & 1);
#endif
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef BLOCKS
            const int blk = it / 16, a = blk & 1;
            const bool first = it % 16 == 0, last = it % 16 == 15;
#else
            const int a = 0;
            const bool first = it == 0, last = false;
#endif
            if (elect_one()) {
                const uint64_t so = (uint64_t)((s * SLOT) >> 4);
                const uint64_t th = dT + so, tl = th + (TAP >> 4), wh = dW + so, wl = wh + (WP >> 4);
                const uint32_t td = tmem + a * NR;
                mma(td, wh, th, idesc, first ? 0u : 1u);
                mma(td, wl, th, idesc, 1u);
                mma(td, wh, tl, idesc, 1u);
                commit(&empty[s]);
                if (last) commit(&accfull[a]);
            }
            __syncwarp();
        }
        if (acc_b == 12345.0) out[0] = 0;
#endif
        // drain: wait for the last items' commits
        for (int it = items - kS; it < items; ++it)
            if (it >= 0) mbar_wait(&empty[it % kS], (it / kS) & 1);
        if ((threadIdx.x & 31) == 0) out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    const int items = 4000, ctas = argc > 1 ? atoi(argv[1]) : 148;
    long long* out;
    CK(cudaMalloc(&out, ctas * 8));
    const int smem = kS * SLOT + 2 * kS * 8 + 32;
    double2* trig;
    CK(cudaMalloc(&trig, 1024 * 16));
    CK(cudaMemset(trig, 0, 1024 * 16));
    CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int rep = 0; rep < 2; ++rep) {
        ring<<<ctas, kThr, smem>>>(items, out, trig);
        CK(cudaDeviceSynchronize());
    }
    long long h[1024];
    CK(cudaMemcpy(h, out, ctas * 8, cudaMemcpyDeviceToHost));
    double m = 0;
    for (int i = 0; i < ctas; ++i) m += (double)h[i] / items;
    printf("{\"variant\": \"%s\", \"ctas\": %d, \"clk_per_item\": %.1f, \"mma_clk_ideal\": 384}\n", VARIANT, ctas, m / ctas);
    return 0;
}

// K1: fused Beer-Lambert + optional Gaussian blur + ramp filter.
//
// Replaces fbp.preprocess (fbp.py:75-83) and fbp.ramp_filter (fbp.py:119-131)
// on the reconstruction path.  The reference zero-pads every (angle, row)
// line to P >= 2n, multiplies its rfft by the real even spectrum of the
// band-limited ramp kernel (fbp.py:86-116) and keeps the first n samples.
// Because the multiplier is real and even, two real lines are filtered by one
// complex FFT (line a in the real part, line b in the imaginary part).  The
// FFT is a shared-memory Stockham transform in persistent CTAs (one line pair
// at a time per CTA), fp32 with fp64-derived twiddles:
//   mode 2 (default, 256 <= P <= 8192): ramp_filter_r8<log2 P>, radix 8, all
//          shapes compile-time, ping-pong buffers, XOR swizzle, prefetch;
//   mode 1 (P = 16384): radix 16 with fused I/O;
//   mode 0 (blur, P < 256): generic passes plus the Gaussian blur.
// Output equals the linear convolution with taps |d| <= n-1 for any pad
// >= 2n, so the transform always runs at next_pow2(2n) whatever
// FilterSpec.padding says.
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.hpp"

struct tf_filter_plan {
    int n;             // channels
    int P;             // internal transform length (pow2 >= 2n)
    int log2P;
    int threads;
    int blur_radius;
    float2* d_tw;      // per-pass twiddle tables (twiddle_tables)
    int n_tw;          // entries
    float* d_mult;     // multiplier / P, m in [0, P/2]
    float* d_blur;     // 2*radius+1 Gaussian weights (or null)
    bool smem_tw;      // twiddles staged in shared memory (P <= 8192)
    int smem;          // dynamic shared memory per CTA
    int max_grid;      // persistent grid: resident CTAs per SM x SMs
    const void* kernel;  // ramp_filter_kernel instantiation for this P
    bool fused;          // fused-I/O FFT path
    int mode;            // 0 generic, 1 fused radix-16, 2 fused radix-8
    int run;             // mode 2: consecutive line pairs per CTA turn (TF_FILTER_RUN)
    double hsum;         // sum |h_P(d)| of the circular kernel K1 applies (incl. 1 / pitch): |T| <= max|x| hsum
};

namespace tf {
namespace {

// ---------------------------------------------------------------- host math
// Band-limited kernel tap at lag d (fbp.py:86-102).
double kernel_tap(int kind, long long d) {
    const double pi2 = M_PI * M_PI;
    if (kind == TF_FILTER_RAMLAK) {
        if (d == 0) return 0.25;
        if (d % 2 == 0) return 0.0;
        return -1.0 / (pi2 * (double)(d * d));
    }
    return -2.0 / (pi2 * (4.0 * (double)d * (double)d - 1.0));
}

// In-place iterative radix-2 complex FFT (fp64), forward sign.
void fft_pow2(std::vector<std::complex<double>>& a) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        for (size_t i = 0; i < n; i += len) {
            for (size_t k = 0; k < len / 2; ++k) {
                double ang = -2.0 * M_PI * (double)k / (double)len;
                std::complex<double> w(cos(ang), sin(ang));
                std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
        }
    }
}

void multiplier_fp64(int kind, long long P, double pitch, double* out) {
    // h on the circular grid (lags m <= P/2 positive, the rest negative)
    std::vector<double> h((size_t)P);
    for (long long m = 0; m < P; ++m) h[(size_t)m] = kernel_tap(kind, m <= P / 2 ? m : m - P);
    const long long nout = P / 2 + 1;
    if ((P & (P - 1)) == 0) {
        std::vector<std::complex<double>> a((size_t)P);
        for (long long m = 0; m < P; ++m) a[(size_t)m] = h[(size_t)m];
        fft_pow2(a);
        for (long long k = 0; k < nout; ++k) out[k] = a[(size_t)k].real() / pitch;
    } else {  // explicit non-pow2 padding: direct real DFT (cos sum) with exact reduction
        for (long long k = 0; k < nout; ++k) {
            double s = 0.0;
            for (long long m = 0; m < P; ++m) {
                long long r = (m * k) % P;
                s += h[(size_t)m] * cos(2.0 * M_PI * (double)r / (double)P);
            }
            out[k] = s / pitch;
        }
    }
}

// ---------------------------------------------------------------- device FFT
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 4); }  // 1 float2 pad per 16

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

// exp(-2 pi i k / 16), k = 0..7
__device__ __forceinline__ float2 w16(int k) {
    constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f, r2 = 0.70710678118654752f;
    switch (k & 7) {
        case 0: return make_float2(1.f, 0.f);
        case 1: return make_float2(c1, -s1);
        case 2: return make_float2(r2, -r2);
        case 3: return make_float2(s1, -c1);
        case 4: return make_float2(0.f, -1.f);
        case 5: return make_float2(-s1, -c1);
        case 6: return make_float2(-r2, -r2);
        default: return make_float2(-c1, -s1);
    }
}

// Forward DFT of R points held in registers (recursive radix-2 DIT; all
// indices are compile-time so everything stays in registers).
template <int R>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
    if constexpr (R == 1) {
        return;
    } else if constexpr (R == 2) {
        float2 a = v[0], b = v[1];
        v[0] = make_float2(a.x + b.x, a.y + b.y);
        v[1] = make_float2(a.x - b.x, a.y - b.y);
    } else {
        constexpr int M = R / 2;
        float2 e[M], o[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            e[i] = v[2 * i];
            o[i] = v[2 * i + 1];
        }
        dft<M>(e);
        dft<M>(o);
#pragma unroll
        for (int k = 0; k < M; ++k) {
            float2 t = (k == 0) ? o[k] : cmul(o[k], w16(k * (16 / R)));
            v[k] = make_float2(e[k].x + t.x, e[k].y + t.y);
            v[k + M] = make_float2(e[k].x - t.x, e[k].y - t.y);
        }
    }
}

// In-place radix-4 DFT of (a, b, c, d) -> (X0, X1, X2, X3), forward sign.
__device__ __forceinline__ void dft4_ip(float2& a, float2& b, float2& c, float2& d) {
    const float2 s0 = make_float2(a.x + c.x, a.y + c.y), d0 = make_float2(a.x - c.x, a.y - c.y);
    const float2 s1 = make_float2(b.x + d.x, b.y + d.y);
    const float2 d1 = make_float2(b.y - d.y, d.x - b.x);  // (b - d) * (-i)
    a = make_float2(s0.x + s1.x, s0.y + s1.y);
    c = make_float2(s0.x - s1.x, s0.y - s1.y);
    b = make_float2(d0.x + d1.x, d0.y + d1.y);
    d = make_float2(d0.x - d1.x, d0.y - d1.y);
}

// In-place radix-16 as 4 x 4 (n = n1 + 4 n2, k = 4 k1 + k2): radix-4 over n2,
// twiddle W16^(n1 k2), radix-4 over n1.  Few temporaries, so a thread keeps
// only its 16 complex values live.  Result X[k] sits at v[dft16_pos(k)].
__host__ __device__ constexpr int dft16_pos(int k) { return 4 * (k % 4) + k / 4; }

__device__ __forceinline__ void dft16_ip(float2 (&v)[16]) {
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4_ip(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
    // now v[n1 + 4 k2] = y[n1][k2]; multiply by W16^(n1 k2)
#pragma unroll
    for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
        for (int k2 = 1; k2 < 4; ++k2) {
            const int e = (n1 * k2) & 15;
            const float2 w = e < 8 ? w16(e) : make_float2(-w16(e - 8).x, -w16(e - 8).y);
            v[n1 + 4 * k2] = cmul(v[n1 + 4 * k2], w);
        }
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) dft4_ip(v[4 * k2], v[4 * k2 + 1], v[4 * k2 + 2], v[4 * k2 + 3]);
    // v[4 k2 + k1] = X[4 k1 + k2]
}

// One Stockham pass of radix R over a padded smem line of length P; each
// thread holds NB radix-R butterflies in registers across the sync.
// IN/OUT select fused I/O so no separate load / multiply / store sweeps
// (and their __syncthreads) are needed:
//   IN_GLOBAL : inputs come from `load(m)` (the first pass; Ns == 1 so inputs
//               r >= R/2 are at m >= P/2 >= n, the zero pad -- pruned);
//   OUT_MULT  : outputs (the natural-order spectrum of the last forward pass)
//               are multiplied by the ramp spectrum / P and conjugated;
//   OUT_GLOBAL: outputs m < n go to `store(m, v)` (the last inverse pass).
// Twiddles `tw` are this pass's [r][k] table (consecutive lanes read
// consecutive entries); with the 1-in-16 padding of pad_idx the radix-16
// passes are bank-conflict-free.
enum { IN_SMEM = 0, IN_GLOBAL = 1 };
enum { OUT_SMEM = 0, OUT_MULT = 1, OUT_GLOBAL = 2 };

template <int R, int NB, int IN, int OUT, class Load, class Store>
__device__ __forceinline__ void fft_pass(float2* buf, const float2* tw, int P, int Ns, int n, int tid, int T,
                                         const Load& load, const float* __restrict__ mult, const Store& store) {
    auto pad = [](int i) { return pad_idx(i); };
    float2 v[NB][R];
    const int nb = P / R;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = tid + b * T;
        if (j < nb) {
            const int k = j & (Ns - 1);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 x;
                if constexpr (IN == IN_GLOBAL) x = (r < R / 2) ? load(j + r * nb) : make_float2(0.f, 0.f);
                else x = buf[pad(j + r * nb)];
                if (r > 0 && Ns > 1) x = cmul(x, tw[r * Ns + k]);
                v[b][r] = x;
            }
            if constexpr (R == 16) dft16_ip(v[b]);
            else dft<R>(v[b]);
        }
    }
    if constexpr (OUT != OUT_GLOBAL) __syncthreads();  // every read of buf done before it is overwritten
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = tid + b * T;
        if (j < nb) {
            const int k = j & (Ns - 1);
            const int base = (j - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int m = base + r * Ns;
                const float2 x = v[b][R == 16 ? dft16_pos(r) : r];
                if constexpr (OUT == OUT_SMEM) {
                    buf[pad(m)] = x;
                } else if constexpr (OUT == OUT_MULT) {
                    // X <- conj(X * M / P): the inverse transform is conj(FFT(conj(.)))
                    const float g = __ldg(&mult[m <= P / 2 ? m : P - m]);
                    buf[pad(m)] = make_float2(x.x * g, -x.y * g);
                } else {
                    if (m < n) store(m, x);
                }
            }
        }
    }
    if constexpr (OUT != OUT_GLOBAL) __syncthreads();
}

// Radix sequences.  Generic path: radix-16 passes, remainder (2/4/8) last.
// Fused radix-16 path (mode 1): radix 16, then the remainder, then radix 16
// -- so the first pass (global input, pruned zero half) and the last pass
// (global output, pruned half) are always radix 16.  Radix-8 path (mode 2):
// 8, remainder, 8, 8, ... (R8Plan mirrors it at compile time).
std::vector<int> radix_plan8(int log2P) {
    std::vector<int> rs{8};
    const int tail = log2P % 3;
    if (tail) rs.push_back(1 << tail);
    for (int i = 1; i < log2P / 3; ++i) rs.push_back(8);
    return rs;
}

std::vector<int> radix_plan(int log2P, bool fused) {
    std::vector<int> rs;
    const int tail = log2P % 4;
    int n16 = log2P / 4;
    if (fused) {
        rs.push_back(16);
        --n16;
        if (tail) rs.push_back(1 << tail);
        for (int i = 0; i < n16; ++i) rs.push_back(16);
    } else {
        for (int i = 0; i < n16; ++i) rs.push_back(16);
        if (tail) rs.push_back(1 << tail);
    }
    return rs;
}

// Per-pass twiddle tables in pass order: for each pass with Ns > 1, R*Ns
// entries [r][k] = exp(-2 pi i k r / (Ns R)) (fp64, rounded once).
std::vector<float2> twiddle_tables(const std::vector<int>& rs) {
    std::vector<float2> t;
    int Ns = 1;
    for (int R : rs) {
        if (Ns > 1)
            for (int r = 0; r < R; ++r)
                for (int k = 0; k < Ns; ++k) {
                    const double a = -2.0 * M_PI * (double)k * (double)r / ((double)Ns * (double)R);
                    t.push_back(make_float2((float)cos(a), (float)sin(a)));
                }
        Ns *= R;
    }
    if (t.empty()) t.push_back(make_float2(1.f, 0.f));
    return t;
}

struct NoIO {
    __device__ float2 operator()(int) const { return make_float2(0.f, 0.f); }
    __device__ void operator()(int, float2) const {}
};

// Generic path: smem -> smem passes only (radix_plan(.., false)).
__device__ __forceinline__ void fft_smem(float2* buf, const float2* tw, int P, int log2P, int tid, int T) {
    const NoIO io;
    int Ns = 1, rem = log2P;
    while (rem >= 4) {
        fft_pass<16, 1, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, P, tid, T, io, nullptr, io);
        if (Ns > 1) tw += 16 * Ns;
        Ns <<= 4;
        rem -= 4;
    }
    if (rem == 3) fft_pass<8, 2, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, P, tid, T, io, nullptr, io);
    else if (rem == 2) fft_pass<4, 4, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, P, tid, T, io, nullptr, io);
    else if (rem == 1) fft_pass<2, 8, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, P, tid, T, io, nullptr, io);
}

// Fused path (radix_plan(.., true), P >= 256): forward with the input load
// and the spectrum multiply folded into its first / last pass, then the
// inverse with the store folded into its last pass.
template <class Load, class Store>
__device__ __forceinline__ void fft_fused(float2* buf, const float2* tw0, int P, int log2P, int n, int tid, int T,
                                          const Load& load, const float* mult, const Store& store) {
    const int tail = log2P % 4;
    const int n16 = log2P / 4;  // >= 2
    for (int dir = 0; dir < 2; ++dir) {
        const float2* tw = tw0;
        int Ns = 1;
        // pass 0: radix 16
        if (dir == 0) fft_pass<16, 1, IN_GLOBAL, OUT_SMEM>(buf, tw, P, Ns, n, tid, T, load, mult, store);
        else fft_pass<16, 1, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, n, tid, T, load, mult, store);
        Ns = 16;
        if (tail) {
            const int R = 1 << tail;
            if (R == 8) fft_pass<8, 2, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, n, tid, T, load, mult, store);
            else if (R == 4) fft_pass<4, 4, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, n, tid, T, load, mult, store);
            else fft_pass<2, 8, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, n, tid, T, load, mult, store);
            tw += R * Ns;
            Ns *= R;
        }
        for (int p = 1; p < n16; ++p) {
            const bool last = p == n16 - 1;
            if (!last) fft_pass<16, 1, IN_SMEM, OUT_SMEM>(buf, tw, P, Ns, n, tid, T, load, mult, store);
            else if (dir == 0) fft_pass<16, 1, IN_SMEM, OUT_MULT>(buf, tw, P, Ns, n, tid, T, load, mult, store);
            else fft_pass<16, 1, IN_SMEM, OUT_GLOBAL>(buf, tw, P, Ns, n, tid, T, load, mult, store);
            tw += 16 * Ns;
            Ns *= 16;
        }
    }
}

// Where filtered line l = (angle a, row r) goes (tf_filter's slab map and
// output layout, see include/tomofuse_b200.h).
struct OutMap {
    int zblocked;        // 0: [a][r][c] rows; 1: z-blocked staging [a][zb][c][36] (K2 input);
                         // 2: K2-TC tap planes [a][hi, lo][r / 8][c][r % 8] fp16 x 2^e[r] (dst[0])
    int n_slabs;         // >= 1 (1 slab == whole row range)
    int rows_per_angle;
    int32_t row0[9];
    float* dst[8];       // start of each slab's block (may be a peer GPU's buffer over NVLink)
    const float* w;      // per-channel feather (z-blocked / tap output only), may be null
    const int* e;        // tap planes: per-row exponents
    int R8;              // tap planes: 8-row groups per angle
};

// Tap-plane destination of line l = (angle a, row r): element offset of (hi plane, channel 0, r % 8)
// and the row's exact scale 2^e[r]
__device__ __forceinline__ __half* taps_ptr(long long l, int n, const OutMap& m, float* dst0, float& sc, int& zi) {
    const long long a = l / m.rows_per_angle;
    const int r = (int)(l - a * m.rows_per_angle);
    zi = r & 7;
    sc = __int_as_float((127 + m.e[r]) << 23);
    return reinterpret_cast<__half*>(dst0) + (a * 2 * m.R8 + (r >> 3)) * (long long)n * 8 + zi;
}

__device__ __forceinline__ void split_half(float x, __half& hi, __half& lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}

// Feathered (fbp.py:242, f32 product), scaled (exact) and split taps of channel m of a line pair:
// both rows in one 4-B store per plane when they share an 8-row group (a even row and its successor)
__device__ __forceinline__ void store_taps(__half* ta, __half* tb, bool has_b, bool pairwise, long long plane8,
                                           int m, float2 y, float wm, float sa, float sb) {
    __half ha, la, hb, lb;
    split_half((y.x * wm) * sa, ha, la);
    if (pairwise) {
        split_half((-y.y * wm) * sb, hb, lb);
        *reinterpret_cast<__half2*>(ta + (size_t)m * 8) = __halves2half2(ha, hb);
        *reinterpret_cast<__half2*>(ta + plane8 + (size_t)m * 8) = __halves2half2(la, lb);
        return;
    }
    ta[(size_t)m * 8] = ha;
    ta[plane8 + (size_t)m * 8] = la;
    if (has_b) {
        split_half((-y.y * wm) * sb, hb, lb);
        tb[(size_t)m * 8] = hb;
        tb[plane8 + (size_t)m * 8] = lb;
    }
}

// row0/base are read from a shared-memory copy (dynamic indexing of a
// kernel-parameter array would spill the struct to local memory)
__device__ __forceinline__ float* out_ptr(long long l, int n, const OutMap& m, const int32_t* row0,
                                          float* const* dst, int& zi) {
    const long long a = l / m.rows_per_angle;
    const int r = (int)(l - a * m.rows_per_angle);
    int s = 0;
#pragma unroll 1
    while (s + 1 < m.n_slabs && r >= row0[s + 1]) ++s;
    const int rl = r - row0[s];
    const int ks = row0[s + 1] - row0[s];
    if (!m.zblocked) {
        zi = 0;
        return dst[s] + (a * ks + rl) * (long long)n;
    }
    const int nzb = (ks + kZB - 1) / kZB;
    zi = rl % kZB;
    return dst[s] + ((a * nzb + rl / kZB) * (long long)n) * kZP + zi;
}

// Persistent: each CTA loops over line pairs; the twiddle table is loaded
// into shared memory once per CTA.
template <bool SMEM_TW, int MAXT, int MODE>
__global__ void __launch_bounds__(MAXT, (MAXT <= 256 ? 2 : 1)) ramp_filter_kernel(const float* __restrict__ in, float* out,
                                                           long long n_lines, int n, int P, int log2P,
                                                           const float2* __restrict__ tw_g,
                                                           const float* __restrict__ mult,
                                                           const float* __restrict__ blur, int radius,
                                                           float i0, OutMap map, int n_tw) {
    extern __shared__ float2 sbuf[];
    __shared__ int32_t s_row0[9];
    __shared__ float* s_dst[8];
    const int tid = threadIdx.x, T = blockDim.x;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < 9; ++s) s_row0[s] = map.row0[s];
#pragma unroll
        for (int s = 0; s < 8; ++s) s_dst[s] = map.dst[s];
    }
    __syncthreads();  // s_row0 / s_dst are read by every thread's out_ptr
    const float2* tw = tw_g;
    float2* data = sbuf;
    if constexpr (SMEM_TW) {
        float2* tws = sbuf + P + P / 16;
        for (int m = tid; m < n_tw; m += T) tws[m] = tw_g[m];
        tw = tws;  // visible after the first __syncthreads below
    }
    const long long n_pairs = (n_lines + 1) / 2;
    const bool log_in = i0 > 0.f;
    for (long long pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
        const long long la = 2 * pair;
        const bool has_b = la + 1 < n_lines;
        const float* pa = in + la * n;
        const float* pb = pa + n;
        // the two lines as one complex line, Beer-Lambert fused (fbp.py:80-83)
        auto load = [&](int m) -> float2 {
            if (m >= n) return make_float2(0.f, 0.f);
            float a = __ldcs(pa + m);
            float b = has_b ? __ldcs(pb + m) : 0.f;
            if (log_in) {  // -ln(max(raw, 1) / i0)
                a = -logf(__fdiv_rn(fmaxf(a, 1.f), i0));
                b = has_b ? -logf(__fdiv_rn(fmaxf(b, 1.f), i0)) : 0.f;
            }
            return make_float2(a, b);
        };
        int za = 0, zb = 0;
        float sa = 1.f, sb = 1.f;
        const bool taps = map.zblocked == 2;
        float* oa = taps ? nullptr : out_ptr(la, n, map, s_row0, s_dst, za);
        float* ob = (has_b && !taps) ? out_ptr(la + 1, n, map, s_row0, s_dst, zb) : nullptr;
        __half* ta = taps ? taps_ptr(la, n, map, s_dst[0], sa, za) : nullptr;
        __half* tb = (taps && has_b) ? taps_ptr(la + 1, n, map, s_dst[0], sb, zb) : nullptr;
        const long long plane8 = (long long)map.R8 * n * 8;
        // both rows in one 8-B (4-B) store when they are z-neighbours of the same block (8-row group)
        const bool pairwise = taps ? (has_b && tb == ta + 1 && (za & 1) == 0)
                                   : (map.zblocked && has_b && (ob == oa + 1) && ((za & 1) == 0));
        auto store = [&](int m, float2 y) {
            if (taps) {
                store_taps(ta, tb, has_b, pairwise, plane8, m, y, map.w ? __ldg(&map.w[m]) : 1.f, sa, sb);
                return;
            }
            if (!map.zblocked) {
                __stcs(oa + m, y.x);
                if (has_b) __stcs(ob + m, -y.y);
                return;
            }
            // feather applied after the filter, as fbp.py:242 does (f32 product)
            const float wm = map.w ? __ldg(&map.w[m]) : 1.f;
            const float va = y.x * wm, vb = -y.y * wm;
            if (pairwise) {
                *reinterpret_cast<float2*>(oa + (size_t)m * kZP) = make_float2(va, vb);
            } else {
                oa[(size_t)m * kZP] = va;
                if (has_b) ob[(size_t)m * kZP] = vb;
            }
        };

        if constexpr (MODE == 1) {
            fft_fused(data, tw, P, log2P, n, tid, T, load, mult, store);
        } else {
            __syncthreads();  // previous pair may still read data[]
            for (int m = tid; m < P; m += T) data[pad_idx(m)] = load(m);
            __syncthreads();
            if (radius > 0) {  // scipy gaussian_filter1d(mode="nearest") restated (fbp.py:125-126)
                float2 acc[8];  // n <= P/2 <= 8*T
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int m = tid + q * T;
                    float2 s = make_float2(0.f, 0.f);
                    if (m < n) {
                        for (int j = -radius; j <= radius; ++j) {
                            const int c = min(max(m + j, 0), n - 1);
                            const float wj = __ldg(&blur[j + radius]);
                            const float2 x = data[pad_idx(c)];
                            s.x = fmaf(wj, x.x, s.x);
                            s.y = fmaf(wj, x.y, s.y);
                        }
                    }
                    acc[q] = s;
                }
                __syncthreads();
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int m = tid + q * T;
                    if (m < n) data[pad_idx(m)] = acc[q];
                }
                __syncthreads();
            }
            fft_smem(data, tw, P, log2P, tid, T);
            // X <- conj(X * M / P): the inverse transform is conj(FFT(conj(.)))
            for (int m = tid; m < P; m += T) {
                const float g = __ldg(&mult[m <= P / 2 ? m : P - m]);
                const float2 x = data[pad_idx(m)];
                data[pad_idx(m)] = make_float2(x.x * g, -x.y * g);
            }
            __syncthreads();
            fft_smem(data, tw, P, log2P, tid, T);
            for (int m = tid; m < n; m += T) store(m, data[pad_idx(m)]);
        }
    }
}

// ----------------------------------------------------------- K1, radix-8 (mode 2)
// Compile-time-shaped variant for 256 <= P <= 8192: T = P/8 threads per line
// pair, one radix-8 butterfly per thread per pass, every stride, twiddle
// offset and buffer a constant.  Two ping-pong line buffers: a pass reads one
// and writes the other, so it needs no barrier between its reads and writes
// and no butterfly value is live across a barrier (64 registers, no spills,
// 2 CTAs x 512 threads per SM at P = 4096).  Instead of padding, an XOR
// swizzle inside each 16-element block,
//     sw8(i) = i ^ ((i >> 4) & 7) ^ (((i >> 6) & 1) << 3),
// maps every radix-8 access pattern of a half-warp (consecutive, stride 8 and
// the 64-blocks of pass 2) onto 16 distinct 8-byte bank pairs.  sw8 is linear
// over GF(2), so for an index a | c with disjoint bit fields
// sw8(a | c) = sw8(a) ^ sw8(c): per butterfly leg sw8(c) is a constant, and
// an immediate address offset wherever it cannot overlap sw8(a)'s bits.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_f2_evict_last(float* p, float a, float b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(a), "f"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_f1_evict_last(float* p, float a, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(a), "l"(pol) : "memory");
}

__host__ __device__ constexpr int sw8(int i) { return i ^ ((i >> 4) & 7) ^ (((i >> 6) & 1) << 3); }

// a_sw = sw8(a) for an index a confined to the bits of `amask`; c a constant
// with bits disjoint from amask
__device__ __forceinline__ int sw8_join(int a_sw, int amask, int c) {
    const int cs = sw8(c);
    return (cs & (amask | 15)) == 0 ? a_sw + cs : a_sw ^ cs;
}

template <int LOG2P>
struct R8Plan {
    static constexpr int P = 1 << LOG2P, T = P / 8, TAIL = LOG2P % 3, N8 = LOG2P / 3, NP = N8 + (TAIL > 0);
    // the pass sequence of radix_plan8: 8, [2^TAIL], 8, 8, ...
    static constexpr int radix(int i) { return i == 0 ? 8 : (TAIL && i == 1) ? (1 << TAIL) : 8; }
    static constexpr int ns(int i) {
        int s = 1;
        for (int q = 0; q < i; ++q) s *= radix(q);
        return s;
    }
    static constexpr int twoff(int i) {  // offset of pass i's [r][k] table in twiddle_tables()
        int o = 0;
        for (int q = 0; q < i; ++q)
            if (ns(q) > 1) o += radix(q) * ns(q);
        return o;
    }
};

// In-place radix-8 (forward sign): X[k] lands in v[(k & 1) * 4 + k / 2].
// HALF: inputs 4..7 are zero (the padded half of the first pass).
template <bool HALF>
__device__ __forceinline__ void dft8_ip(float2 (&v)[8]) {
    constexpr float r2 = 0.70710678118654752f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if constexpr (HALF) {
            v[k + 4] = v[k];
        } else {
            const float2 a = v[k], b = v[k + 4];
            v[k] = make_float2(a.x + b.x, a.y + b.y);
            v[k + 4] = make_float2(a.x - b.x, a.y - b.y);
        }
    }
    // odd half times W8^k: W8 = (1 - i)/sqrt2, W8^2 = -i, W8^3 = -(1 + i)/sqrt2
    {
        const float2 b = v[5];
        v[5] = make_float2((b.x + b.y) * r2, (b.y - b.x) * r2);
    }
    v[6] = make_float2(v[6].y, -v[6].x);
    {
        const float2 b = v[7];
        v[7] = make_float2((b.y - b.x) * r2, -(b.x + b.y) * r2);
    }
    dft4_ip(v[0], v[1], v[2], v[3]);  // X0 X2 X4 X6
    dft4_ip(v[4], v[5], v[6], v[7]);  // X1 X3 X5 X7
}
__host__ __device__ constexpr int dft8_pos(int k) { return (k & 1) * 4 + k / 2; }

// One Stockham pass (radix R, input stride NS) of a P-point line: src -> dst.
// FULL: n == P/2 (power-of-two line length), so every first-pass input leg is
// inside the line and exactly the last pass's legs r < R/2 are stored.
template <int LOG2P, int R, int NS, int IN, int OUT, bool FULL, class Load, class Store>
__device__ __forceinline__ void r8_pass(const float2* src, float2* dst, const float2* tw, int tid, int n,
                                        const Load& load, const float* __restrict__ mult, const Store& store) {
    constexpr int P = 1 << LOG2P, T = P / 8, NB = 8 / R, STRIDE = P / R;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = tid + b * T;  // butterfly, < P/R
        float2 v[R];
        const int j_sw = sw8(j);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if constexpr (IN == IN_GLOBAL) {
                v[r] = r < R / 2 ? load(r, j + r * STRIDE) : make_float2(0.f, 0.f);
            } else {
                v[r] = src[sw8_join(j_sw, STRIDE - 1, r * STRIDE)];
            }
        }
        const int k = j & (NS - 1);
        if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * NS + k]);
        }
        if constexpr (R == 8) {
            if constexpr (IN == IN_GLOBAL) dft8_ip<true>(v);
            else dft8_ip<false>(v);
        } else if constexpr (R == 4) {
            dft4_ip(v[0], v[1], v[2], v[3]);
        } else {
            const float2 a = v[0], c = v[1];
            v[0] = make_float2(a.x + c.x, a.y + c.y);
            v[1] = make_float2(a.x - c.x, a.y - c.y);
        }
        const int base = (j - k) * R + k;
        const int b_sw = sw8(base);
        constexpr int BMASK = (P - 1) & ~((NS * R - 1) & ~(NS - 1));  // bits base may occupy
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float2 x = v[R == 8 ? dft8_pos(r) : r];
            if constexpr (OUT == OUT_SMEM) {
                dst[sw8_join(b_sw, BMASK, r * NS)] = x;
            } else if constexpr (OUT == OUT_MULT) {
                // X <- conj(X * M / P): the inverse transform is conj(FFT(conj(.)))
                const int m = base + r * NS;
                const float g = __ldg(&mult[m <= P / 2 ? m : P - m]);
                dst[sw8_join(b_sw, BMASK, r * NS)] = make_float2(x.x * g, -x.y * g);
            } else {
                const int m = base + r * NS;
                if (FULL ? r < R / 2 : m < n) store(m, x);
            }
        }
    }
}

// Passes I.. of one direction; pass G = DIR * NP + I writes buffer G % 2.
template <int LOG2P, int I, int DIR, bool FULL, class Load, class Store>
__device__ __forceinline__ void r8_run(float2* bufs, const float2* tw, int tid, int n, const Load& load,
                                       const float* mult, const Store& store) {
    using PL = R8Plan<LOG2P>;
    if constexpr (I < PL::NP) {
        constexpr int G = DIR * PL::NP + I;
        constexpr int IN = (DIR == 0 && I == 0) ? IN_GLOBAL : IN_SMEM;
        constexpr int OUT = I == PL::NP - 1 ? (DIR == 0 ? OUT_MULT : OUT_GLOBAL) : OUT_SMEM;
        r8_pass<LOG2P, PL::radix(I), PL::ns(I), IN, OUT, FULL>(bufs + ((G + 1) % 2) * PL::P,
                                                               bufs + (G % 2) * PL::P, tw + PL::twoff(I), tid, n,
                                                               load, mult, store);
        if constexpr (OUT != OUT_GLOBAL) __syncthreads();
        r8_run<LOG2P, I + 1, DIR, FULL>(bufs, tw, tid, n, load, mult, store);
    }
}

// The persistent line-pair loop of ramp_filter_r8.
template <int LOG2P, bool FULL>
__device__ __forceinline__ void r8_pairs(const float* __restrict__ in, long long n_lines, int n,
                                         const float* __restrict__ mult, float i0, const OutMap& map, int run,
                                         float2* sbuf, const float2* tws, const int32_t* s_row0,
                                         float* const* s_dst) {
    constexpr int P = 1 << LOG2P;
    const int tid = threadIdx.x;
    const long long n_pairs = (n_lines + 1) / 2;
    const bool log_in = i0 > 0.f;
    const float inv_i0 = 1.f / i0;
    const NoIO none;
    const uint64_t pol = policy_evict_last();
    // raw inputs of this thread's 4 first-pass legs (m = tid + r P/8, r < 4),
    // loaded one pair ahead so the loads overlap the previous pair's inverse
    float2 pf[4];
    auto prefetch = [&](long long pr) {
        if (pr >= n_pairs) return;
        const long long l = 2 * pr;
        const float* pa = in + l * n;
        const bool hb = l + 1 < n_lines;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int m = tid + r * (P / 8);
            pf[r] = make_float2(0.f, 0.f);
            if (FULL || m < n) pf[r] = make_float2(__ldcs(pa + m), hb ? __ldcs(pa + n + m) : 0.f);
        }
    };
    // CTA b takes runs of kRun consecutive line pairs: pairs kRun*(b + i*grid) + j.
    // Consecutive pairs are neighbouring rows of one z-block, so one CTA
    // completes each 32-B staging sector (8 rows of a channel) within a few
    // pairs instead of 4 CTAs scattering 8-B pieces of it across L2.
    const int kRun = run;
    auto pair_of = [&](long long it) { return kRun * (blockIdx.x + (it / kRun) * gridDim.x) + it % kRun; };
    prefetch(pair_of(0));
    for (long long it = 0;; ++it) {
        const long long pair = pair_of(it);
        if (pair >= n_pairs) {
            if (it % kRun == 0) break;  // past the end
            continue;                   // ragged last run
        }
        const long long la = 2 * pair;
        const bool has_b = la + 1 < n_lines;
        {
            // the two lines as one complex line, Beer-Lambert fused (fbp.py:80-83)
            auto load = [&](int r, int m) -> float2 {
                if (!FULL && m >= n) return make_float2(0.f, 0.f);
                float a = pf[r].x, b = pf[r].y;
                if (log_in) {  // -ln(max(raw, 1) / i0)
                    // MUFU.LG2-based log of the ratio (in (0, 1]): |error| < 4e-7 for
                    // ratios in [0.5, 1], ~1 ulp relative below -- far inside the fp32
                    // filter's own error, and 8 logs per thread per pair were ~8% of
                    // K1's instructions with the polynomial logf
                    a = -__logf(fmaxf(a, 1.f) * inv_i0);
                    b = has_b ? -__logf(fmaxf(b, 1.f) * inv_i0) : 0.f;
                }
                return make_float2(a, b);
            };
            __syncthreads();  // the previous pair's last pass may still read buffer 0
            r8_run<LOG2P, 0, 0, FULL>(sbuf, tws, tid, n, load, mult, none);
        }
        prefetch(pair_of(it + 1) < n_pairs ? pair_of(it + 1) : pair_of(it + kRun - it % kRun));
        // output pointers resolved after the forward half (fewer live registers)
        int za = 0, zb = 0;
        float sa = 1.f, sb = 1.f;
        const bool taps = map.zblocked == 2;
        float* oa = taps ? nullptr : out_ptr(la, n, map, s_row0, s_dst, za);
        float* ob = (has_b && !taps) ? out_ptr(la + 1, n, map, s_row0, s_dst, zb) : nullptr;
        __half* ta = taps ? taps_ptr(la, n, map, s_dst[0], sa, za) : nullptr;
        __half* tb = (taps && has_b) ? taps_ptr(la + 1, n, map, s_dst[0], sb, zb) : nullptr;
        const long long plane8 = (long long)map.R8 * n * 8;
        // both rows in one 8-B (4-B) store when they are z-neighbours of the same block (8-row group)
        const bool pairwise = taps ? (has_b && tb == ta + 1 && (za & 1) == 0)
                                   : (map.zblocked && has_b && (ob == oa + 1) && ((za & 1) == 0));
        const float* w = map.w;
        const bool zbl = map.zblocked;
        auto store = [&](int m, float2 y) {
            if (taps) {
                store_taps(ta, tb, has_b, pairwise, plane8, m, y, w ? __ldg(&w[m]) : 1.f, sa, sb);
                return;
            }
            if (!zbl) {
                __stcs(oa + m, y.x);
                if (has_b) __stcs(ob + m, -y.y);
                return;
            }
            const float wm = w ? __ldg(&w[m]) : 1.f;  // feather after the filter (fbp.py:242)
            const float va = y.x * wm, vb = -y.y * wm;
            // evict_last: a staging line is completed by 16 line pairs; keep the
            // partial line in L2 until then (the raw input streams evict-first)
            if (pairwise) {
                st_f2_evict_last(oa + (size_t)m * kZP, va, vb, pol);
            } else {
                st_f1_evict_last(oa + (size_t)m * kZP, va, pol);
                if (has_b) st_f1_evict_last(ob + (size_t)m * kZP, vb, pol);
            }
        };
        r8_run<LOG2P, 0, 1, FULL>(sbuf, tws, tid, n, none, mult, store);
    }
}

// Same arguments as ramp_filter_kernel (blur/radius unused: no blur in mode 2).
template <int LOG2P>
__global__ void __launch_bounds__(R8Plan<LOG2P>::T, 1024 / R8Plan<LOG2P>::T)
    ramp_filter_r8(const float* __restrict__ in, float* out, long long n_lines, int n, int, int,
                   const float2* __restrict__ tw_g, const float* __restrict__ mult, const float* __restrict__,
                   int run, float i0, OutMap map, int n_tw) {  // `run` rides in ramp_filter_kernel's blur-radius slot
    constexpr int P = 1 << LOG2P;
    extern __shared__ float2 sbuf[];  // [2][P] ping-pong lines, then the twiddle tables
    __shared__ int32_t s_row0[9];
    __shared__ float* s_dst[8];
    const int tid = threadIdx.x;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < 9; ++s) s_row0[s] = map.row0[s];
#pragma unroll
        for (int s = 0; s < 8; ++s) s_dst[s] = map.dst[s];
    }
    float2* tws = sbuf + 2 * P;
    for (int m = tid; m < n_tw; m += R8Plan<LOG2P>::T) tws[m] = tw_g[m];
    __syncthreads();
    if (2 * n == P) r8_pairs<LOG2P, true>(in, n_lines, n, mult, i0, map, run, sbuf, tws, s_row0, s_dst);
    else r8_pairs<LOG2P, false>(in, n_lines, n, mult, i0, map, run, sbuf, tws, s_row0, s_dst);
}

template <typename T>
__global__ void preprocess_kernel(const T* __restrict__ raw, double* __restrict__ out, long long n, double i0) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long step = (long long)gridDim.x * blockDim.x;
    for (; i < n; i += step) {
        double c = fmax((double)raw[i], 1.0);  // LOG_CLAMP_COUNTS, fbp.py:26
        out[i] = -log(__ddiv_rn(c, i0));
    }
}

}  // namespace
}  // namespace tf

using namespace tf;

extern "C" int tf_filter_multiplier(int kind, int64_t padded, double pixel_pitch, double* host_out) {
    if (kind != TF_FILTER_RAMLAK && kind != TF_FILTER_SHEPPLOGAN)
        return set_error(TF_ERR_INVALID_ARGUMENT, "unknown filter kind %d", kind);
    if (padded < 1 || !(pixel_pitch > 0) || !host_out)
        return set_error(TF_ERR_INVALID_ARGUMENT, "invalid multiplier arguments");
    multiplier_fp64(kind, padded, pixel_pitch, host_out);
    return TF_OK;
}

extern "C" int tf_filter_plan_create(int n_chan, int kind, int64_t padded, double pixel_pitch,
                                     double blur_sigma, tf_filter_plan** plan) {
    if (!plan) return set_error(TF_ERR_INVALID_ARGUMENT, "null plan pointer");
    *plan = nullptr;
    if (kind != TF_FILTER_RAMLAK && kind != TF_FILTER_SHEPPLOGAN)
        return set_error(TF_ERR_INVALID_ARGUMENT, "unknown filter kind %d", kind);
    if (n_chan < 1) return set_error(TF_ERR_INVALID_ARGUMENT, "n_chan must be >= 1");
    if (blur_sigma < 0) return set_error(TF_ERR_INVALID_ARGUMENT, "blur_sigma must be >= 0");
    if (!(pixel_pitch > 0)) return set_error(TF_ERR_INVALID_ARGUMENT, "pixel_pitch must be positive");
    const long long need = 2LL * n_chan;
    if (padded != 0 && padded < need)  // FilterSpec.padded_length, fbp.py:50-55
        return set_error(TF_ERR_INVALID_ARGUMENT, "padding %lld below required %lld for %d channels",
                         (long long)padded, need, n_chan);
    int P = 1;
    while (P < need) P <<= 1;
    if (P > 16 * 1024) return set_error(TF_ERR_UNSUPPORTED, "n_chan %d exceeds the 8192-channel filter kernel", n_chan);
    auto* p = new tf_filter_plan();
    p->n = n_chan;
    p->P = P;
    p->log2P = ilog2(P);
    p->threads = std::max(32, P / 16);  // one radix-16 butterfly per thread (P <= 16384 -> <= 1024)
    // K1 variant: radix-8 ramp_filter_r8 (256 <= P <= 8192), fused radix-16
    // (P = 16384 or TF_FILTER_MODE=1), generic smem path (blur, P < 256)
    const char* fm = getenv("TF_FILTER_MODE");
    p->mode = blur_sigma > 0 ? 0 : (P >= 256 && P <= 8192 ? 2 : (p->log2P >= 8 ? 1 : 0));
    if (fm && blur_sigma <= 0) {
        const int want = atoi(fm);
        if (want == 0 || (want == 1 && p->log2P >= 8) || (want == 2 && P >= 256 && P <= 8192)) p->mode = want;
    }
    p->fused = p->mode != 0;
    const char* fr = getenv("TF_FILTER_RUN");
    p->run = fr ? std::max(1, std::min(64, atoi(fr))) : 8;
    if (p->mode == 2) p->threads = std::max(32, P / 8);
    std::vector<float2> tw =
        twiddle_tables(p->mode == 2 ? radix_plan8(p->log2P) : radix_plan(p->log2P, p->mode == 1));
    p->n_tw = (int)tw.size();
    std::vector<double> mult(P / 2 + 1);
    multiplier_fp64(kind, P, pixel_pitch, mult.data());
    std::vector<float> multf(P / 2 + 1);
    for (int k = 0; k <= P / 2; ++k) multf[k] = (float)(mult[k] / (double)P);
    {
        // the spatial kernel K1 applies is h_P = IFFT(multiplier) (real, even): its l1 norm bounds
        // |filtered| by max|input| (the blur is a normalised non-negative kernel)
        std::vector<std::complex<double>> X((size_t)P);
        for (int k = 0; k < P; ++k) X[(size_t)k] = mult[(size_t)(k <= P / 2 ? k : P - k)];
        fft_pow2(X);
        double hs = 0;
        for (int k = 0; k < P; ++k) hs += std::fabs(X[(size_t)k].real()) / (double)P;
        p->hsum = hs;
    }
    int rad = 0;
    std::vector<float> bw;
    if (blur_sigma > 0) {  // scipy: radius = int(truncate * sigma + 0.5), truncate 4
        rad = (int)(4.0 * blur_sigma + 0.5);
        std::vector<double> w(2 * rad + 1);
        double sum = 0;
        for (int j = -rad; j <= rad; ++j) {
            w[j + rad] = exp(-0.5 / (blur_sigma * blur_sigma) * (double)j * (double)j);
            sum += w[j + rad];
        }
        bw.resize(2 * rad + 1);
        for (int j = 0; j <= 2 * rad; ++j) bw[j] = (float)(w[j] / sum);
    }
    p->blur_radius = rad;
    cudaError_t e = cudaMalloc(&p->d_tw, sizeof(float2) * p->n_tw);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_mult, sizeof(float) * (P / 2 + 1));
    if (e == cudaSuccess && rad > 0) e = cudaMalloc(&p->d_blur, sizeof(float) * (2 * rad + 1));
    if (e == cudaSuccess) e = cudaMemcpy(p->d_tw, tw.data(), sizeof(float2) * p->n_tw, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_mult, multf.data(), sizeof(float) * (P / 2 + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && rad > 0)
        e = cudaMemcpy(p->d_blur, bw.data(), sizeof(float) * (2 * rad + 1), cudaMemcpyHostToDevice);
    p->smem_tw = P <= 8192;  // twiddle table in shared memory next to the line buffer
    p->smem = ((p->mode == 2 ? 2 * P : P + P / 16) + (p->smem_tw ? p->n_tw : 0)) * (int)sizeof(float2);
    if (p->mode == 2) {
        switch (p->log2P) {
            case 8: p->kernel = (const void*)ramp_filter_r8<8>; break;
            case 9: p->kernel = (const void*)ramp_filter_r8<9>; break;
            case 10: p->kernel = (const void*)ramp_filter_r8<10>; break;
            case 11: p->kernel = (const void*)ramp_filter_r8<11>; break;
            case 12: p->kernel = (const void*)ramp_filter_r8<12>; break;
            default: p->kernel = (const void*)ramp_filter_r8<13>; break;
        }
    } else if (p->mode == 1)
        p->kernel = p->threads <= 256 ? (const void*)ramp_filter_kernel<true, 256, 1>
                    : p->threads <= 512 ? (const void*)ramp_filter_kernel<true, 512, 1>
                                        : (const void*)ramp_filter_kernel<false, 1024, 1>;
    else
        p->kernel = p->threads <= 256 ? (const void*)ramp_filter_kernel<true, 256, 0>
                    : p->threads <= 512 ? (const void*)ramp_filter_kernel<true, 512, 0>
                                        : (const void*)ramp_filter_kernel<false, 1024, 0>;
    // the attribute is per-function global state shared by every plan: raise it
    // to the device's opt-in maximum (never lower it to this plan's size)
    if (e == cudaSuccess) {
        int dev = 0, optin = 0;
        e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa{};
        if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, p->kernel);
        const int maxdyn = optin - (int)fa.sharedSizeBytes;  // static smem counts against the opt-in limit
        if (e == cudaSuccess && p->smem > maxdyn) e = cudaErrorInvalidValue;
        if (e == cudaSuccess) e = cudaFuncSetAttribute(p->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, maxdyn);
    }
    if (e == cudaSuccess) {
        int blocks = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, p->kernel, p->threads, p->smem);
        int dev = 0, sms = 148;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        p->max_grid = std::max(1, blocks) * sms;
    }
    if (e != cudaSuccess) {
        tf_filter_plan_destroy(p);
        return set_error(TF_ERR_CUDA, "filter plan setup failed: %s", cudaGetErrorString(e));
    }
    *plan = p;
    return TF_OK;
}

extern "C" int tf_filter_plan_destroy(tf_filter_plan* p) {
    if (!p) return TF_OK;
    cudaFree(p->d_tw);
    cudaFree(p->d_mult);
    cudaFree(p->d_blur);
    delete p;
    return TF_OK;
}

namespace tf {
namespace {
int build_map(OutMap& map, float* out, int64_t n_lines, int rows_per_angle, int n_slabs, const int32_t* slab_row0,
              const int64_t* slab_base, void* const* slab_dst = nullptr) {
    map.n_slabs = n_slabs > 0 ? n_slabs : 1;
    map.rows_per_angle = rows_per_angle > 0 ? rows_per_angle : (int)std::min<int64_t>(n_lines, 1 << 30);
    if (n_slabs > 0) {
        if (n_slabs > 8 || rows_per_angle < 1 || !slab_row0 || (!slab_base && !slab_dst))
            return set_error(TF_ERR_INVALID_ARGUMENT, "invalid slab map");
        for (int s = 0; s <= n_slabs; ++s) map.row0[s] = slab_row0[s];
        for (int s = 0; s < n_slabs; ++s) {
            map.dst[s] = slab_dst ? static_cast<float*>(slab_dst[s]) : out + slab_base[s];
            if (!map.dst[s]) return set_error(TF_ERR_INVALID_ARGUMENT, "null slab destination");
        }
        if (map.row0[0] != 0 || map.row0[n_slabs] != rows_per_angle)
            return set_error(TF_ERR_INVALID_ARGUMENT, "slab rows must cover [0, rows_per_angle)");
        for (int s = 0; s < n_slabs; ++s)
            if (map.row0[s + 1] < map.row0[s]) return set_error(TF_ERR_INVALID_ARGUMENT, "slab rows must ascend");
    } else {
        map.row0[0] = 0;
        map.row0[1] = map.rows_per_angle;
        map.dst[0] = out;
    }
    if (rows_per_angle > 0 && n_lines % rows_per_angle != 0)
        return set_error(TF_ERR_INVALID_ARGUMENT, "n_lines must be a multiple of rows_per_angle");
    return TF_OK;
}

int launch_filter(const tf_filter_plan* p, const float* in, float* out, int64_t n_lines, float i0,
                  const OutMap& map, void* stream) {
    const long long pairs = (n_lines + 1) / 2;
    const long long units = p->mode == 2 ? (pairs + p->run - 1) / p->run : pairs;  // r8: runs of `run` pairs
    const unsigned grid = (unsigned)std::min<long long>(units, p->max_grid);
    long long nl = n_lines;
    int n = p->n, P = p->P, l2 = p->log2P, rad = p->mode == 2 ? p->run : p->blur_radius;
    const float2* tw = p->d_tw;
    const float* mult = p->d_mult;
    const float* blur = p->d_blur;
    OutMap m = map;
    int ntw = p->n_tw;
    void* args[] = {(void*)&in, (void*)&out, &nl, &n, &P, &l2, (void*)&tw, (void*)&mult, (void*)&blur, &rad,
                    &i0, &m, &ntw};
    TF_CUDA_TRY(cudaLaunchKernel(p->kernel, dim3(grid), dim3(p->threads), args, p->smem, as_stream(stream)));
    return TF_OK;
}
}  // namespace
}  // namespace tf

extern "C" int tf_filter(const tf_filter_plan* p, const float* in, float* out, int64_t n_lines, float i0,
                         int rows_per_angle, int n_slabs, const int32_t* slab_row0, const int64_t* slab_base,
                         void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null filter plan");
    if (n_lines < 0) return set_error(TF_ERR_INVALID_ARGUMENT, "n_lines must be >= 0");
    if (n_lines == 0) return TF_OK;
    if (!in || !out) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    if (n_slabs > 0 && in == out) return set_error(TF_ERR_INVALID_ARGUMENT, "slab-major output cannot be in place");
    OutMap map{};
    int st = build_map(map, out, n_lines, n_slabs > 0 ? rows_per_angle : 0, n_slabs, slab_row0, slab_base);
    if (st) return st;
    map.zblocked = 0;
    map.w = nullptr;
    return launch_filter(p, in, out, n_lines, i0, map, stream);
}

extern "C" int tf_filter_stage(const tf_filter_plan* p, const tf_bp_plan* bp, const float* in, void* stage,
                               int64_t n_lines, float i0, int rows_per_angle, int n_slabs,
                               const int32_t* slab_row0, const int64_t* slab_base, void* stream) {
    if (!p || !bp) return set_error(TF_ERR_INVALID_ARGUMENT, "null plan");
    if (n_lines < 0 || rows_per_angle < 1) return set_error(TF_ERR_INVALID_ARGUMENT, "invalid line counts");
    if (n_lines == 0) return TF_OK;
    if (!in || !stage) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    if (bp_plan_n_chan(bp) != p->n) return set_error(TF_ERR_INVALID_ARGUMENT, "filter/bp plans disagree on n_chan");
    OutMap map{};
    int st = build_map(map, static_cast<float*>(stage), n_lines, rows_per_angle, n_slabs, slab_row0, slab_base);
    if (st) return st;
    map.zblocked = 1;
    map.w = bp_plan_weights(bp);
    return launch_filter(p, in, static_cast<float*>(stage), n_lines, i0, map, stream);
}

extern "C" int tf_filter_stage_peers(const tf_filter_plan* p, const tf_bp_plan* bp, const float* in,
                                     int64_t n_lines, float i0, int rows_per_angle, int n_slabs,
                                     const int32_t* slab_row0, void* const* slab_dst, void* stream) {
    if (!p || !bp) return set_error(TF_ERR_INVALID_ARGUMENT, "null plan");
    if (n_lines < 0 || rows_per_angle < 1 || n_slabs < 1) return set_error(TF_ERR_INVALID_ARGUMENT, "invalid line counts");
    if (n_lines == 0) return TF_OK;
    if (!in || !slab_dst) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    if (bp_plan_n_chan(bp) != p->n) return set_error(TF_ERR_INVALID_ARGUMENT, "filter/bp plans disagree on n_chan");
    OutMap map{};
    int st = build_map(map, nullptr, n_lines, rows_per_angle, n_slabs, slab_row0, nullptr, slab_dst);
    if (st) return st;
    map.zblocked = 1;
    map.w = bp_plan_weights(bp);
    return launch_filter(p, in, map.dst[0], n_lines, i0, map, stream);
}

extern "C" int tf_filter_peers(const tf_filter_plan* p, const float* in, int64_t n_lines, float i0,
                               int rows_per_angle, int n_slabs, const int32_t* slab_row0, void* const* slab_dst,
                               void* stream) {
    if (!p) return set_error(TF_ERR_INVALID_ARGUMENT, "null plan");
    if (n_lines < 0 || rows_per_angle < 1 || n_slabs < 1) return set_error(TF_ERR_INVALID_ARGUMENT, "invalid line counts");
    if (n_lines == 0) return TF_OK;
    if (!in || !slab_dst) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    OutMap map{};
    int st = build_map(map, nullptr, n_lines, rows_per_angle, n_slabs, slab_row0, nullptr, slab_dst);
    if (st) return st;
    map.zblocked = 0;  // natural rows: each line one contiguous run (coalesced NVLink stores)
    map.w = nullptr;
    return launch_filter(p, in, map.dst[0], n_lines, i0, map, stream);
}

namespace tf {
namespace {
// |depth| = |ln i0 - ln max(raw, 1)| <= max(|ln i0|, |ln i0 - ln FLT_MAX|) for finite counts
double depth_bound(double i0) {
    const double l = std::log(i0);
    return std::max(std::fabs(l), std::fabs(l - std::log(3.4028234663852886e38)));
}
constexpr double kTapMargin = 1.01;  // fp32 FFT round-off above the exact l1 bound
}  // namespace
}  // namespace tf

extern "C" int tf_filter_tap_bound(const tf_filter_plan* p, double i0, double* bound) {
    if (!p || !bound) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    if (!(i0 > 0)) return set_error(TF_ERR_INVALID_ARGUMENT, "i0 must be positive, got %g", i0);
    *bound = depth_bound(i0) * p->hsum * kTapMargin;
    return TF_OK;
}

extern "C" int tf_filter_taps(const tf_filter_plan* p, const tf_bp_plan* bp, const float* in, void* taps,
                              int64_t taps_bytes, int64_t n_lines, float i0, int rows_per_angle, void* stream) {
    if (!p || !bp) return set_error(TF_ERR_INVALID_ARGUMENT, "null plan");
    if (n_lines < 0 || rows_per_angle < 1) return set_error(TF_ERR_INVALID_ARGUMENT, "invalid line counts");
    if (n_lines % rows_per_angle != 0)
        return set_error(TF_ERR_INVALID_ARGUMENT, "n_lines must be a multiple of rows_per_angle");
    if (bp_plan_n_chan(bp) != p->n) return set_error(TF_ERR_INVALID_ARGUMENT, "filter/bp plans disagree on n_chan");
    if (!tf_bp_tc_supported(bp))
        return set_error(TF_ERR_UNSUPPORTED, "tensor-core tap planes need voxel_pitch / pixel_pitch <= 2.12");
    if (!in || !taps) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    const int n_ang = (int)(n_lines / rows_per_angle);
    const int64_t need = tf_bp_tc_taps_bytes(bp, rows_per_angle, n_ang);
    if (taps_bytes < need)
        return set_error(TF_ERR_INVALID_ARGUMENT, "tap workspace too small: %lld < %lld bytes", (long long)taps_bytes,
                         (long long)need);
    cudaStream_t s = as_stream(stream);
    int st = i0 > 0.f ? tc_uniform_exponents(taps, rows_per_angle, depth_bound(i0) * p->hsum * kTapMargin, s)
                      : tc_row_exponents(taps, in, rows_per_angle, n_ang, p->n, nullptr, p->hsum * kTapMargin, s);
    if (st) return st;
    if (n_lines == 0) return TF_OK;
    OutMap map{};
    st = build_map(map, reinterpret_cast<float*>(static_cast<uint8_t*>(taps) + bp_tc_header_bytes(bp, rows_per_angle)),
                   n_lines, rows_per_angle, 0, nullptr, nullptr);
    if (st) return st;
    map.zblocked = 2;
    map.w = bp_plan_weights(bp);
    map.e = static_cast<const int*>(taps);
    map.R8 = (rows_per_angle + 7) / 8;
    return launch_filter(p, in, map.dst[0], n_lines, i0, map, stream);
}

extern "C" int tf_preprocess(const void* raw, int raw_dtype, double* out, int64_t n, double i0, void* stream) {
    if (!(i0 > 0)) return set_error(TF_ERR_INVALID_ARGUMENT, "i0 must be positive, got %g", i0);
    if (n < 0 || (raw_dtype != TF_F32 && raw_dtype != TF_F64)) return set_error(TF_ERR_INVALID_ARGUMENT, "bad arguments");
    if (n == 0) return TF_OK;
    if (!raw || !out) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (raw_dtype == TF_F32)
        preprocess_kernel<float><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const float*>(raw), out, n, i0);
    else
        preprocess_kernel<double><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const double*>(raw), out, n, i0);
    return check_launch("preprocess_kernel");
}

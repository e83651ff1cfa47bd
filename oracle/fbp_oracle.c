/*
 * CPU oracle for the FBP hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference back-projection and filter
 * (/root/reference/pkg/src/tomofuse/fbp.py + geometry.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg load it, through
 * ctypes, as the checker.  The product library never links it.
 *
 * Compiled with -ffp-contract=off (no FMA contraction) so the float64 path is
 * bit-identical to the reference's numpy float64 arithmetic:
 *   t   = ((x-cx)*cos(th) + (y-cy)*sin(th)) * scale + axis   geometry.py:148-153
 *   th  = k * (span / n_proj)                               geometry.py:69-70
 *   acc += line[c0]*w0 + line[c1]*w1 (ascending k)          fbp.py:233-245
 *   FoV zeroing, then * (span/n_proj)                        fbp.py:246-251
 * and the float32 path mirrors numpy's float32 promotion of the same
 * expressions (frac cast to f32, line*weights in f32, f32 accumulate).
 * tests/test_cpu_host.py (the oracle-vs-golden tests) pins both against reference-generated vectors.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

/* Minimal dynamic parallel-for over [0, n) on pthreads (libgomp is absent
 * from this image).  Rows / lines are independent, so scheduling never
 * changes any result. */
typedef void (*body_fn)(long i, void *ctx);
typedef struct {
    body_fn fn;
    void *ctx;
    long n;
    long next;
    pthread_mutex_t mu;
} pfor_t;

static void *pfor_worker(void *arg) {
    pfor_t *p = (pfor_t *)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        long i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->n) break;
        p->fn(i, p->ctx);
    }
    return NULL;
}

static void parallel_for(long n, int n_threads, body_fn fn, void *ctx) {
    pfor_t p;
    p.fn = fn;
    p.ctx = ctx;
    p.n = n;
    p.next = 0;
    pthread_mutex_init(&p.mu, NULL);
    int nt = n_threads > 1 ? n_threads : 1;
    if (nt > 256) nt = 256;
    pthread_t th[256];
    for (int i = 1; i < nt; i++) pthread_create(&th[i], NULL, pfor_worker, &p);
    pfor_worker(&p);
    for (int i = 1; i < nt; i++) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&p.mu);
}

/* fbp.py:147-183 */
static void feather(double *w, int n, int offset_chan, int band) {
    int i;
    if (offset_chan == 0) {
        for (i = 0; i < n; i++) w[i] = 1.0;
        return;
    }
    double c0 = (n - 1) / 2.0 - offset_chan;
    for (i = 0; i < n; i++) {
        double c = (double)i;
        double near = offset_chan > 0 ? c : (double)(n - 1) - c;
        double own = near / band;
        own = own < 0.0 ? 0.0 : (own > 1.0 ? 1.0 : own);
        double m = 2.0 * c0 - c;
        double other = 0.0;
        if (m >= 0 && m <= n - 1) {
            double mn = offset_chan > 0 ? m : (double)(n - 1) - m;
            other = mn / band;
            other = other < 0.0 ? 0.0 : (other > 1.0 ? 1.0 : other);
        }
        double tot = own + other;
        w[i] = tot > 0 ? own / tot : 0.0;
    }
}

void oracle_offset_weights(double *w, int n, int offset_chan, int band) {
    feather(w, n, offset_chan, band);
}

typedef struct {
    const double *sino;
    const double *w;
    double *out;
    int n_proj, n_rows, n_chan, nx, ny, a0, a1, x0, x1, y0, y1, use_f32;
    int n_bands, band;  /* work unit = (detector row, band of `band` image rows) */
    double step, cx, cy, sc, axis, R2, sc2;
} bp_ctx;

/* One detector row == one volume slice (geometry.py:134-139); a work unit is
 * one slice's band of image rows [y0 + b*band, ...), so a single slice also
 * spreads over the threads.  Every voxel still sums its angles in ascending
 * order exactly as fbp.py:233-245, so the split does not change any bit. */
static void bp_row(long u, void *vctx) {
    const bp_ctx *g0 = (const bp_ctx *)vctx;
    const long r = u / g0->n_bands;
    bp_ctx gb = *g0;
    gb.y0 = g0->y0 + (int)(u % g0->n_bands) * g0->band;
    gb.y1 = gb.y0 + g0->band < g0->y1 ? gb.y0 + g0->band : g0->y1;
    const bp_ctx *g = &gb;
    int n = g->n_chan, tw = g->x1 - g->x0, th = g->y1 - g->y0;
    size_t plane = (size_t)g->nx * g->ny;
    double *acc = (double *)calloc((size_t)tw * th, sizeof(double));
    float *accf = (float *)calloc((size_t)tw * th, sizeof(float));
    float *linef = (float *)malloc(sizeof(float) * n);
    double *lined = (double *)malloc(sizeof(double) * n);
    for (int k = g->a0; k < g->a1; k++) {
        double ang = (double)k * g->step;
        double cs = cos(ang), sn = sin(ang);
        const double *src = g->sino + ((size_t)k * g->n_rows + r) * n;
        for (int c = 0; c < n; c++) {
            lined[c] = src[c] * g->w[c];
            linef[c] = (float)src[c] * (float)g->w[c];
        }
        for (int yy = 0; yy < th; yy++) {
            double ty = ((double)(g->y0 + yy) - g->cy) * sn;
            for (int xx = 0; xx < tw; xx++) {
                double t = ((double)(g->x0 + xx) - g->cx) * cs;
                t = t + ty;
                t = t * g->sc + g->axis;
                int64_t lo = (int64_t)floor(t);
                int ok0 = lo >= 0 && lo < n;
                int ok1 = lo + 1 >= 0 && lo + 1 < n;
                int64_t c0 = ok0 ? lo : 0, c1 = ok1 ? lo + 1 : 0;
                size_t o = (size_t)yy * tw + xx;
                if (g->use_f32) {
                    float f = (float)(t - (double)lo);
                    float w0 = ok0 ? 1.0f - f : 0.0f;
                    float w1 = ok1 ? f : 0.0f;
                    float g0 = linef[c0] * w0;
                    float g1 = linef[c1] * w1;
                    accf[o] = accf[o] + (g0 + g1);
                } else {
                    double f = t - (double)lo;
                    double w0 = ok0 ? 1.0 - f : 0.0;
                    double w1 = ok1 ? f : 0.0;
                    double g0 = lined[c0] * w0;
                    double g1 = lined[c1] * w1;
                    acc[o] = acc[o] + (g0 + g1);
                }
            }
        }
    }
    float awf = (float)g->step;
    for (int yy = 0; yy < th; yy++) {
        double dy = (double)(g->y0 + yy) - g->cy;
        for (int xx = 0; xx < tw; xx++) {
            double dx = (double)(g->x0 + xx) - g->cx;
            double rr = (dx * dx + dy * dy) * g->sc2;
            size_t o = (size_t)yy * tw + xx;
            double v;
            if (rr > g->R2)
                v = 0.0;
            else if (g->use_f32)
                v = (double)(accf[o] * awf);
            else
                v = acc[o] * g->step;
            g->out[(size_t)r * plane + (size_t)(g->y0 + yy) * g->nx + (g->x0 + xx)] = v;
        }
    }
    free(acc);
    free(accf);
    free(linef);
    free(lined);
}

/* sino: (n_proj, n_rows, n_chan) float64 holding the selected rows only;
 * out:  (n_rows, ny, nx) float64 (float32 results widened when use_f32). */
int oracle_back_project(const double *sino, int n_proj, int n_rows, int n_chan,
                        int nx, int ny, double span, double pixel_pitch,
                        double voxel_pitch, int offset_chan, int a0, int a1,
                        int x0, int x1, int y0, int y1, int feather_band,
                        int use_f32, double *out, int n_threads) {
    size_t plane = (size_t)nx * ny;
    memset(out, 0, sizeof(double) * plane * (size_t)n_rows);
    if (n_rows == 0 || a1 == a0 || x1 == x0 || y1 == y0) return 0;
    if (offset_chan != 0 && feather_band < 1) return -1;
    double *w = (double *)malloc(sizeof(double) * n_chan);
    feather(w, n_chan, offset_chan, feather_band);
    bp_ctx g;
    g.sino = sino;
    g.w = w;
    g.out = out;
    g.n_proj = n_proj; g.n_rows = n_rows; g.n_chan = n_chan;
    g.nx = nx; g.ny = ny; g.a0 = a0; g.a1 = a1;
    g.x0 = x0; g.x1 = x1; g.y0 = y0; g.y1 = y1; g.use_f32 = use_f32;
    g.step = span / n_proj;
    g.cx = (nx - 1) / 2.0;
    g.cy = (ny - 1) / 2.0;
    g.sc = voxel_pitch / pixel_pitch;
    g.axis = (n_chan - 1) / 2.0 - offset_chan;
    double half = (n_chan - 1) / 2.0;
    double R = offset_chan != 0 ? half + fabs((double)offset_chan) : half;
    g.R2 = R * R;
    g.sc2 = g.sc * g.sc;
    /* enough units for the threads even for one slice: bands of >= 16 image rows */
    int nt = n_threads > 0 ? n_threads : 1;
    int want = (4 * nt + n_rows - 1) / n_rows;
    g.band = (y1 - y0 + want - 1) / want;
    if (g.band < 16) g.band = 16;
    g.n_bands = (y1 - y0 + g.band - 1) / g.band;
    parallel_for((long)n_rows * g.n_bands, n_threads, bp_row, &g);
    free(w);
    return 0;
}

/* fbp.py:86-102 */
static double tap(int kind, long d) {
    double pi2 = M_PI * M_PI;
    if (kind == 0) {
        if (d == 0) return 0.25;
        if (d % 2 == 0) return 0.0;
        return -1.0 / (pi2 * (double)(d * d));
    }
    return -2.0 / (pi2 * (4.0 * (double)d * (double)d - 1.0));
}

/* fbp.py:75-83 */
void oracle_preprocess(const double *raw, double *out, long n, double i0) {
    for (long i = 0; i < n; i++) {
        double c = raw[i] > 1.0 ? raw[i] : 1.0;
        out[i] = -log(c / i0);
    }
}

/* fbp.py:119-131 restated as the equivalent linear convolution with taps
 * |d| <= n-1 (exact because the pad is >= 2n); optional scipy-style
 * gaussian_filter1d(mode="nearest") first.  kind 0 = ramlak, 1 = shepplogan. */
typedef struct {
    const double *in;
    double *out;
    const double *taps;
    const double *gw;
    int n, rad;
    double pitch;
} flt_ctx;

static void flt_line(long l, void *vctx) {
    const flt_ctx *g = (const flt_ctx *)vctx;
    int n = g->n;
    const double *x = g->in + l * n;
    double *buf = (double *)malloc(sizeof(double) * n);
    if (g->rad > 0) {
        for (int i = 0; i < n; i++) {
            double s = 0;
            for (int j = -g->rad; j <= g->rad; j++) {
                int c = i + j;
                c = c < 0 ? 0 : (c > n - 1 ? n - 1 : c);
                s += g->gw[j + g->rad] * x[c];
            }
            buf[i] = s;
        }
    } else {
        memcpy(buf, x, sizeof(double) * n);
    }
    for (int i = 0; i < n; i++) {
        double s = 0;
        for (int j = 0; j < n; j++) s += buf[j] * g->taps[i - j + n - 1];
        g->out[l * n + i] = s / g->pitch;
    }
    free(buf);
}

/* fbp.py:119-131 restated as the equivalent linear convolution with taps
 * |d| <= n-1 (exact because the pad is >= 2n); optional scipy-style
 * gaussian_filter1d(mode="nearest") first.  kind 0 = ramlak, 1 = shepplogan. */
void oracle_ramp_filter(const double *in, double *out, long n_lines, int n,
                        int kind, double pixel_pitch, double blur_sigma,
                        int n_threads) {
    double *taps = (double *)malloc(sizeof(double) * (2 * (size_t)n - 1));
    for (long d = -(n - 1); d <= n - 1; d++) taps[d + n - 1] = tap(kind, d);
    int rad = 0;
    double *gw = NULL;
    if (blur_sigma > 0) {
        rad = (int)(4.0 * blur_sigma + 0.5);
        gw = (double *)malloc(sizeof(double) * (2 * (size_t)rad + 1));
        double sum = 0;
        for (int j = -rad; j <= rad; j++) {
            gw[j + rad] = exp(-0.5 / (blur_sigma * blur_sigma) * (double)j * (double)j);
            sum += gw[j + rad];
        }
        for (int j = 0; j <= 2 * rad; j++) gw[j] /= sum;
    }
    flt_ctx g;
    g.in = in;
    g.out = out;
    g.taps = taps;
    g.gw = gw;
    g.n = n;
    g.rad = rad;
    g.pitch = pixel_pitch;
    parallel_for(n_lines, n_threads, flt_line, &g);
    free(taps);
    free(gw);
}

/* fbp.py:255-259 (np.round == round-half-even == nearbyint in FE_TONEAREST) */
void oracle_quantize(const double *v, uint16_t *q, long n, double lo, double hi) {
    for (long i = 0; i < n; i++) {
        double s = (v[i] - lo) / (hi - lo);
        s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
        q[i] = (uint16_t)nearbyint(s * 65535.0);
    }
}

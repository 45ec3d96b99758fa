/*
 * CPU restatement of the reference forward + render_target, T = float.
 * TEST INFRASTRUCTURE ONLY — see lvs_oracle.h. Each function cites the
 * reference file:line (relative to /root/reference/proj) whose arithmetic it
 * restates. Built with -ffp-contract=off like the reference
 * (CMakeLists.txt:11-15): every a*b+c below rounds twice.
 */
#define _GNU_SOURCE
#include "lvs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* threading: split independent outputs; never changes per-output order      */
/* ------------------------------------------------------------------------ */

static int g_threads = 0;

void lvso_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

static int nthreads(void) {
  if (g_threads > 0) return g_threads;
  const char* e = getenv("LVSO_THREADS");
  int n = e ? atoi(e) : 1;
  return n < 1 ? 1 : n;
}

typedef void (*range_fn)(void* ctx, int64_t b, int64_t e);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t b, e;
} job_t;

static void* job_run(void* p) {
  job_t* j = (job_t*)p;
  if (j->b < j->e) j->fn(j->ctx, j->b, j->e);
  return NULL;
}

static void par_for(int64_t n, range_fn fn, void* ctx) {
  int t = nthreads();
  if (t > n) t = (int)(n > 0 ? n : 1);
  if (t <= 1) {
    if (n > 0) fn(ctx, 0, n);
    return;
  }
  pthread_t th[256];
  job_t jobs[256];
  if (t > 256) t = 256;
  for (int i = 0; i < t; ++i) {
    jobs[i].fn = fn;
    jobs[i].ctx = ctx;
    jobs[i].b = n * i / t;
    jobs[i].e = n * (i + 1) / t;
  }
  for (int i = 1; i < t; ++i) pthread_create(&th[i], NULL, job_run, &jobs[i]);
  job_run(&jobs[0]);
  for (int i = 1; i < t; ++i) pthread_join(th[i], NULL);
}

static float* falloc(int64_t n) {
  float* p = (float*)calloc((size_t)(n > 0 ? n : 1), sizeof(float));
  if (!p) {
    fprintf(stderr, "lvs_oracle: out of memory (%lld floats)\n", (long long)n);
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------------ */
/* scalar kernels (kernels_ref.hpp)                                          */
/* ------------------------------------------------------------------------ */

/* dot_blocked: 8 lane accumulators, fixed combine tree (kernels_ref.hpp:15-25). */
static float dot_blocked(const float* a, const float* b, int64_t n) {
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t i = 0;
  for (; i + 8 <= n; i += 8)
    for (int j = 0; j < 8; ++j) acc[j] += a[i + j] * b[i + j];
  for (; i < n; ++i) acc[i & 7] += a[i] * b[i];
  float s01 = acc[0] + acc[1], s23 = acc[2] + acc[3];
  float s45 = acc[4] + acc[5], s67 = acc[6] + acc[7];
  return (s01 + s23) + (s45 + s67);
}

/* matmul: C[M,N] = A[M,K] B[K,N], k ascending from 0 (kernels_ref.hpp:40-48). */
typedef struct {
  const float *A, *B;
  float* C;
  int64_t K, N;
} mm_ctx;

static void mm_rows(void* p, int64_t b, int64_t e) {
  mm_ctx* c = (mm_ctx*)p;
  const int64_t K = c->K, N = c->N;
  for (int64_t m = b; m < e; ++m) {
    float* out = c->C + m * N;
    for (int64_t n = 0; n < N; ++n) out[n] = 0.f;
    for (int64_t k = 0; k < K; ++k) {
      float a = c->A[m * K + k];
      const float* brow = c->B + k * N;
      for (int64_t n = 0; n < N; ++n) out[n] += a * brow[n];
    }
  }
}

static void matmul(const float* A, const float* B, float* C, int64_t M, int64_t K, int64_t N) {
  mm_ctx c = {A, B, C, K, N};
  par_for(M, mm_rows, &c);
}

/* conv3x3 (kernels_ref.hpp:61-96): acc starts at bias, taps ci, di, dj
 * ascending, out-of-bounds taps skipped. Vectorised over j with the same
 * per-output order (as kernels_avx2.cpp:80-107 does). */
typedef struct {
  const float *x, *w, *b;
  float* y;
  int64_t Cin, Cout, H, W;
} conv_ctx;

static void conv_rows(void* p, int64_t b, int64_t e) {
  conv_ctx* c = (conv_ctx*)p;
  const int64_t Cin = c->Cin, H = c->H, W = c->W;
  for (int64_t r = b; r < e; ++r) {
    int64_t co = r / H, i = r % H;
    float* y = c->y + (co * H + i) * W;
    float bias = c->b ? c->b[co] : 0.f;
    for (int64_t j = 0; j < W; ++j) y[j] = bias;
    for (int64_t ci = 0; ci < Cin; ++ci)
      for (int64_t di = 0; di < 3; ++di) {
        int64_t ii = i + di - 1;
        if (ii < 0 || ii >= H) continue;
        const float* xr = c->x + (ci * H + ii) * W;
        const float* wr = c->w + ((co * Cin + ci) * 3 + di) * 3;
        for (int64_t dj = 0; dj < 3; ++dj) {
          float wv = wr[dj];
          int64_t lo = dj == 0 ? 1 : 0;
          int64_t hi = dj == 2 ? W - 1 : W;
          const float* xs = xr + dj - 1;
          for (int64_t j = lo; j < hi; ++j) y[j] += wv * xs[j];
        }
      }
  }
}

void lvso_conv3x3(const float* x, const float* w, const float* b, float* y, int64_t Cin,
                  int64_t Cout, int64_t H, int64_t W) {
  conv_ctx c = {x, w, b, y, Cin, Cout, H, W};
  par_for(Cout * H, conv_rows, &c);
}

/* ------------------------------------------------------------------------ */
/* elementwise semantics (tape.hpp)                                          */
/* ------------------------------------------------------------------------ */

/* gelu, exact erf form (tape.hpp:313-319). */
static inline float gelu(float x) {
  const float inv_sqrt2 = (float)0.70710678118654752440;
  return 0.5f * x * (1.0f + erff(x * inv_sqrt2));
}
/* sigmoid (tape.hpp:284-288). */
static inline float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }

/* activate_depth_from_logits (ldm.hpp:73-83): tanh, scale T(0.5/L), + anchor,
 * scale T(1/near-1/far), offset T(1/far), recip. */
static inline float depth_act(float x, int64_t l, int64_t L, float s1, float s2, float s3) {
  float anchor = (float)(((double)l + 0.5) / (double)L);
  float t = tanhf(x) * s1;
  float dn = t + anchor;
  float disp = dn * s2 + s3;
  return 1.0f / disp;
}

/* rms_norm (tape.hpp:771-787): one row of C. */
static inline void rms_row(const float* x, const float* g, float* out, int64_t C) {
  float ms = 0.f;
  for (int64_t c = 0; c < C; ++c) ms += x[c] * x[c];
  ms /= (float)C;
  float r = 1.0f / sqrtf(ms + (float)1e-6);
  for (int64_t c = 0; c < C; ++c) out[c] = x[c] * r * g[c];
}

/* resize_bilinear taps (tape.hpp:866-881). */
typedef struct {
  int64_t* i0;
  int64_t* i1;
  float* f;
} taps_t;

static taps_t make_taps(int64_t out_n, int64_t in_n) {
  taps_t t;
  t.i0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)out_n);
  t.i1 = (int64_t*)malloc(sizeof(int64_t) * (size_t)out_n);
  t.f = (float*)malloc(sizeof(float) * (size_t)out_n);
  double s = (double)in_n / (double)out_n;
  for (int64_t i = 0; i < out_n; ++i) {
    double u = ((double)i + 0.5) * s - 0.5;
    double fl = floor(u);
    int64_t a = (int64_t)fl;
    t.f[i] = (float)(u - fl);
    int64_t a0 = a < 0 ? 0 : (a > in_n - 1 ? in_n - 1 : a);
    int64_t a1 = a + 1 < 0 ? 0 : (a + 1 > in_n - 1 ? in_n - 1 : a + 1);
    t.i0[i] = a0;
    t.i1[i] = a1;
  }
  return t;
}

static void free_taps(taps_t t) {
  free(t.i0);
  free(t.i1);
  free(t.f);
}

/* resize_bilinear over planes [B,H,W] -> [B,Ho,Wo] (tape.hpp:884-896). */
static void resize_planes(const float* src, float* dst, int64_t B, int64_t H, int64_t W,
                          int64_t Ho, int64_t Wo) {
  if (H == Ho && W == Wo) {
    memcpy(dst, src, sizeof(float) * (size_t)(B * H * W));
    return;
  }
  taps_t ty = make_taps(Ho, H), tx = make_taps(Wo, W);
  for (int64_t n = 0; n < B; ++n) {
    const float* s = src + n * H * W;
    float* d = dst + n * Ho * Wo;
    for (int64_t i = 0; i < Ho; ++i)
      for (int64_t j = 0; j < Wo; ++j) {
        float a = s[ty.i0[i] * W + tx.i0[j]], b = s[ty.i0[i] * W + tx.i1[j]];
        float c = s[ty.i1[i] * W + tx.i0[j]], e = s[ty.i1[i] * W + tx.i1[j]];
        float top = a + (b - a) * tx.f[j];
        float bot = c + (e - c) * tx.f[j];
        d[i * Wo + j] = top + (bot - top) * ty.f[i];
      }
  }
  free_taps(ty);
  free_taps(tx);
}

/* resize of channel-last maps [B,H,W,C] via the reference's
 * hwc_to_chw -> resize -> chw_to_hwc (identical per-channel arithmetic). */
static void resize_hwc(const float* src, float* dst, int64_t B, int64_t H, int64_t W, int64_t C,
                       int64_t Ho, int64_t Wo) {
  if (H == Ho && W == Wo) {
    memcpy(dst, src, sizeof(float) * (size_t)(B * H * W * C));
    return;
  }
  taps_t ty = make_taps(Ho, H), tx = make_taps(Wo, W);
  for (int64_t n = 0; n < B; ++n) {
    const float* s = src + n * H * W * C;
    float* d = dst + n * Ho * Wo * C;
    for (int64_t i = 0; i < Ho; ++i)
      for (int64_t j = 0; j < Wo; ++j)
        for (int64_t c = 0; c < C; ++c) {
          float a = s[(ty.i0[i] * W + tx.i0[j]) * C + c], b = s[(ty.i0[i] * W + tx.i1[j]) * C + c];
          float cc = s[(ty.i1[i] * W + tx.i0[j]) * C + c], e = s[(ty.i1[i] * W + tx.i1[j]) * C + c];
          float top = a + (b - a) * tx.f[j];
          float bot = cc + (e - cc) * tx.f[j];
          d[(i * Wo + j) * C + c] = top + (bot - top) * ty.f[i];
        }
  }
  free_taps(ty);
  free_taps(tx);
}

static void hwc_to_chw(const float* src, float* dst, int64_t H, int64_t W, int64_t C) {
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j)
      for (int64_t c = 0; c < C; ++c) dst[(c * H + i) * W + j] = src[(i * W + j) * C + c];
}
static void chw_to_hwc(const float* src, float* dst, int64_t H, int64_t W, int64_t C) {
  for (int64_t c = 0; c < C; ++c)
    for (int64_t i = 0; i < H; ++i)
      for (int64_t j = 0; j < W; ++j) dst[(i * W + j) * C + c] = src[(c * H + i) * W + j];
}

/* over_composite (ldm.hpp:98-115): o = v*a + (1-a)*o, l ascending from 0. */
static void over_composite(const float* v, const float* s, float* out, int64_t L, int64_t P,
                           int64_t C) {
  memset(out, 0, sizeof(float) * (size_t)(P * C));
  for (int64_t p = 0; p < P; ++p)
    for (int64_t l = 0; l < L; ++l) {
      float a = s[l * P + p];
      const float* vl = v + (l * P + p) * C;
      float* o = out + p * C;
      for (int64_t c = 0; c < C; ++c) o[c] = vl[c] * a + (1.0f - a) * o[c];
    }
}

/* ------------------------------------------------------------------------ */
/* cameras and geometry (camera.cpp, geometry.hpp)                           */
/* ------------------------------------------------------------------------ */

/* Camera::scaled (camera.cpp:67-78). */
static lvsg_camera cam_scaled(const lvsg_camera* c, int64_t nw, int64_t nh) {
  lvsg_camera o = *c;
  double sx = (double)nw / (double)c->width;
  double sy = (double)nh / (double)c->height;
  o.fx = c->fx * sx;
  o.cx = c->cx * sx;
  o.fy = c->fy * sy;
  o.cy = c->cy * sy;
  o.width = nw;
  o.height = nh;
  return o;
}

typedef struct {
  double R[9], t[3], fx, fy, cx, cy;
  int64_t W, H;
} campod;

/* CamPod::from (geometry.hpp:18-32). */
static campod pod(const lvsg_camera* c) {
  campod p;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) p.R[i * 3 + j] = c->cam_from_world[i * 4 + j];
    p.t[i] = c->cam_from_world[i * 4 + 3];
  }
  p.fx = c->fx;
  p.fy = c->fy;
  p.cx = c->cx;
  p.cy = c->cy;
  p.W = c->width;
  p.H = c->height;
  return p;
}

/* Camera::center = -R^T t with the shim's k-ascending product
 * (camera.cpp:40-49). */
static void cam_center(const lvsg_camera* c, double out[3]) {
  const double* m = c->cam_from_world;
  for (int r = 0; r < 3; ++r) {
    double acc = (-m[0 * 4 + r]) * m[0 * 4 + 3];
    acc += (-m[1 * 4 + r]) * m[1 * 4 + 3];
    acc += (-m[2 * 4 + r]) * m[2 * 4 + 3];
    out[r] = acc;
  }
}

/* R^T * ray_dir_cam(u, v) (camera.cpp:51-53; geometry.hpp:97). */
static void world_dir(const lvsg_camera* c, double u, double v, double out[3]) {
  const double* m = c->cam_from_world;
  double d0 = (u - c->cx) / c->fx, d1 = (v - c->cy) / c->fy, d2 = 1.0;
  for (int r = 0; r < 3; ++r) {
    double acc = m[0 * 4 + r] * d0;
    acc += m[1 * 4 + r] * d1;
    acc += m[2 * 4 + r] * d2;
    out[r] = acc;
  }
}

/* world_points (geometry.hpp:84-129); returns 1 on out-of-range depth. */
int lvso_world_points(const lvsg_frustum* fr, const float* depth, int64_t L, int64_t H, int64_t W,
                      float* out) {
  lvsg_camera cam = cam_scaled(&fr->camera, W, H);
  double c[3];
  cam_center(&cam, c);
  double* dirs = (double*)malloc(sizeof(double) * (size_t)(H * W * 3));
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) world_dir(&cam, (double)j + 0.5, (double)i + 0.5, dirs + (i * W + j) * 3);
  double slack = 1e-3 * (fr->far_depth - fr->near_depth);
  int bad = 0;
  for (int64_t l = 0; l < L; ++l)
    for (int64_t p = 0; p < H * W; ++p) {
      double dv = (double)depth[l * H * W + p];
      if (dv < fr->near_depth - slack || dv > fr->far_depth + slack) bad = 1;
      for (int k = 0; k < 3; ++k) out[(l * H * W + p) * 3 + k] = (float)(dv * dirs[p * 3 + k] + c[k]);
    }
  free(dirs);
  return bad;
}

typedef struct {
  int64_t x0, x1, y0, y1;
  double fx, fy;
  int valid;
} fp_t;

/* footprint (geometry.hpp:58-79). */
static inline fp_t footprint(double u, double v, int64_t W, int64_t H) {
  fp_t f;
  const double tol = 1e-4;
  f.valid = u >= 0.5 - tol && u <= (double)W - 0.5 + tol && v >= 0.5 - tol &&
            v <= (double)H - 0.5 + tol;
  if (!f.valid) {
    f.x0 = f.x1 = f.y0 = f.y1 = 0;
    f.fx = f.fy = 0;
    return f;
  }
  u = fmin(fmax(u, 0.5), (double)W - 0.5);
  v = fmin(fmax(v, 0.5), (double)H - 0.5);
  double xf = floor(u - 0.5), yf = floor(v - 0.5);
  f.x0 = (int64_t)xf;
  f.y0 = (int64_t)yf;
  f.fx = u - 0.5 - xf;
  f.fy = v - 0.5 - yf;
  f.x1 = f.x0 + 1 < W - 1 ? f.x0 + 1 : W - 1;
  f.y1 = f.y0 + 1 < H - 1 ? f.y0 + 1 : H - 1;
  return f;
}

/* Validity-margin trace (parity attribution): with
 * lvso_trace_margins enabled, every footprint the forward computes in a
 * gather (backproject_stack) or a splat (render_to_input_view) whose
 * projected point lies within `tol` pixels of its validity boundary is
 * recorded as one row of 8 floats: step, kind (0 gather, 1 splat), view,
 * layer, y, x (texel of that step's volume), signed margin in pixels
 * (> 0 inside), coordinate (u or v) that sets it. Observation only: the
 * arithmetic and the results are unchanged. */
static float* g_tr_buf = NULL;
static int64_t g_tr_cap = 0, g_tr_n = 0, g_tr_H = 1, g_tr_W = 1;
static double g_tr_tol = 0.0;
static int g_tr_step = -1, g_tr_kind = 0, g_tr_view = 0;
static pthread_mutex_t g_tr_mu = PTHREAD_MUTEX_INITIALIZER;

void lvso_trace_margins(double tol, float* buf, int64_t cap) {
  g_tr_tol = tol;
  g_tr_buf = buf;
  g_tr_cap = buf ? cap : 0;
  g_tr_n = 0;
}
int64_t lvso_trace_count(void) { return g_tr_n; }

static void trace_ctx(int step, int kind, int view, int64_t H, int64_t W) {
  g_tr_step = step;
  g_tr_kind = kind;
  g_tr_view = view;
  g_tr_H = H;
  g_tr_W = W;
}

static inline void trace_uv(int64_t texel, double u, double v, int64_t Wi, int64_t Hi) {
  if (!g_tr_buf) return;
  const double tol = 1e-4;
  const double m[4] = {u - (0.5 - tol), ((double)Wi - 0.5 + tol) - u, v - (0.5 - tol),
                       ((double)Hi - 0.5 + tol) - v};
  int a = 0;
  for (int i = 1; i < 4; ++i)
    if (fabs(m[i]) < fabs(m[a])) a = i;
  if (fabs(m[a]) >= g_tr_tol) return;
  pthread_mutex_lock(&g_tr_mu);
  if (g_tr_n < g_tr_cap) {
    float* r = g_tr_buf + g_tr_n * 8;
    const int64_t plane = g_tr_H * g_tr_W, q = texel % plane;
    r[0] = (float)g_tr_step;
    r[1] = (float)g_tr_kind;
    r[2] = (float)g_tr_view;
    r[3] = (float)(texel / plane);
    r[4] = (float)(q / g_tr_W);
    r[5] = (float)(q % g_tr_W);
    r[6] = (float)m[a];
    r[7] = (float)(a < 2 ? u : v);
  }
  g_tr_n++;
  pthread_mutex_unlock(&g_tr_mu);
}

/* CamPod::to_cam + projection + footprint (geometry.hpp:34-37, :152-159). */
static inline fp_t project_fp_t(const campod* cp, const float* pt, int64_t texel) {
  double pw[3] = {(double)pt[0], (double)pt[1], (double)pt[2]};
  double q[3];
  for (int i = 0; i < 3; ++i)
    q[i] = cp->R[i * 3 + 0] * pw[0] + cp->R[i * 3 + 1] * pw[1] + cp->R[i * 3 + 2] * pw[2] + cp->t[i];
  fp_t f;
  if (q[2] <= 1e-6) {
    memset(&f, 0, sizeof(f));
    return f;
  }
  double u = cp->fx * q[0] / q[2] + cp->cx;
  double v = cp->fy * q[1] / q[2] + cp->cy;
  trace_uv(texel, u, v, cp->W, cp->H);
  return footprint(u, v, cp->W, cp->H);
}

static inline fp_t project_fp(const campod* cp, const float* pt) {
  double pw[3] = {(double)pt[0], (double)pt[1], (double)pt[2]};
  double q[3];
  for (int i = 0; i < 3; ++i)
    q[i] = cp->R[i * 3 + 0] * pw[0] + cp->R[i * 3 + 1] * pw[1] + cp->R[i * 3 + 2] * pw[2] + cp->t[i];
  fp_t f;
  if (q[2] <= 1e-6) {
    memset(&f, 0, sizeof(f));
    return f;
  }
  double u = cp->fx * q[0] / q[2] + cp->cx;
  double v = cp->fy * q[1] / q[2] + cp->cy;
  return footprint(u, v, cp->W, cp->H);
}

void lvso_footprints(const lvsg_camera* cam, const float* points, int64_t P, int32_t* taps,
                     uint8_t* valid, double* fracs) {
  campod cp = pod(cam);
  for (int64_t p = 0; p < P; ++p) {
    fp_t f = project_fp(&cp, points + p * 3);
    taps[p * 4 + 0] = (int32_t)f.x0;
    taps[p * 4 + 1] = (int32_t)f.x1;
    taps[p * 4 + 2] = (int32_t)f.y0;
    taps[p * 4 + 3] = (int32_t)f.y1;
    valid[p] = (uint8_t)f.valid;
    fracs[p * 2] = f.fx;
    fracs[p * 2 + 1] = f.fy;
  }
}

/* gather_backproject (geometry.hpp:138-171): f64 blend, cast to T. Output
 * row stride `ostride` lets backproject_stack write [..,M,C] in place. */
typedef struct {
  campod cp;
  const float* img;
  int64_t Hi, Wi, C;
  const float* pts;
  float* out;
  int64_t ostride;
  float* mask;
  int64_t mstride;
  int traced;
} gather_ctx;

static void gather_rows(void* p, int64_t b, int64_t e) {
  gather_ctx* g = (gather_ctx*)p;
  const int64_t C = g->C, Wi = g->Wi;
  for (int64_t i = b; i < e; ++i) {
    fp_t f = g->traced ? project_fp_t(&g->cp, g->pts + i * 3, i) : project_fp(&g->cp, g->pts + i * 3);
    float* o = g->out + i * g->ostride;
    if (!f.valid) {
      for (int64_t c = 0; c < C; ++c) o[c] = 0.f;
      if (g->mask) g->mask[i * g->mstride] = 0.f;
      continue;
    }
    if (g->mask) g->mask[i * g->mstride] = 1.f;
    double w00 = (1 - f.fx) * (1 - f.fy), w10 = f.fx * (1 - f.fy);
    double w01 = (1 - f.fx) * f.fy, w11 = f.fx * f.fy;
    const float* i00 = g->img + (f.y0 * Wi + f.x0) * C;
    const float* i10 = g->img + (f.y0 * Wi + f.x1) * C;
    const float* i01 = g->img + (f.y1 * Wi + f.x0) * C;
    const float* i11 = g->img + (f.y1 * Wi + f.x1) * C;
    for (int64_t c = 0; c < C; ++c)
      o[c] = (float)(w00 * (double)i00[c] + w10 * (double)i10[c] + w01 * (double)i01[c] +
                     w11 * (double)i11[c]);
  }
}

static void gather_strided(const lvsg_camera* cam, const float* image, int64_t Hi, int64_t Wi,
                           int64_t C, const float* points, int64_t P, float* values,
                           int64_t ostride, float* mask, int64_t mstride) {
  gather_ctx g = {pod(cam), image, Hi, Wi, C, points, values, ostride, mask, mstride, 0};
  par_for(P, gather_rows, &g);
}

void lvso_gather(const lvsg_camera* cam, const float* image, int64_t Hi, int64_t Wi, int64_t C,
                 const float* points, int64_t P, float* values, float* mask) {
  gather_strided(cam, image, Hi, Wi, C, points, P, values, C, mask, 1);
}

/* backproject_stack (network.hpp:421-436): Δ [P, M, C]. */
static void backproject_stack(float* const* feats, const lvsg_camera* ucams, int64_t M,
                              int64_t Hf, int64_t Wf, int64_t C, const float* pts, int64_t P,
                              float* deltas) {
  for (int64_t m = 0; m < M; ++m) {
    gather_ctx g = {pod(&ucams[m]), feats[m], Hf, Wf, C, pts, deltas + m * C, M * C, NULL, 0,
                    g_tr_buf != NULL};
    g_tr_kind = 0;
    g_tr_view = (int)m;
    par_for(P, gather_rows, &g);
  }
}

/* splat_accumulate + splat_project (geometry.hpp:230-264, :317-326):
 * values [L,H,W,K] -> normalised [L,Hi,Wi,K]. Sequential (l, texel) order. */
static void splat_project(const float* val, const float* pts, int64_t L, int64_t H, int64_t W,
                          int64_t K, const lvsg_camera* cam, float* out) {
  campod cp = pod(cam);
  const int64_t Hi = cam->height, Wi = cam->width, PL = H * W;
  float* acc = falloc(L * Hi * Wi * (K + 1));
  for (int64_t l = 0; l < L; ++l)
    for (int64_t s = 0; s < PL; ++s) {
      int64_t p = l * PL + s;
      fp_t f = project_fp_t(&cp, pts + p * 3, p);
      if (!f.valid) continue;
      double w[4] = {(1 - f.fx) * (1 - f.fy), f.fx * (1 - f.fy), (1 - f.fx) * f.fy, f.fx * f.fy};
      int64_t tap[4] = {(l * Hi + f.y0) * Wi + f.x0, (l * Hi + f.y0) * Wi + f.x1,
                        (l * Hi + f.y1) * Wi + f.x0, (l * Hi + f.y1) * Wi + f.x1};
      for (int k = 0; k < 4; ++k) {
        float* dst = acc + tap[k] * (K + 1);
        float wk = (float)w[k];
        for (int64_t c = 0; c < K; ++c) dst[c] += wk * val[p * K + c];
        dst[K] += wk;
      }
    }
  const float eps = (float)1e-4;
  for (int64_t q = 0; q < L * Hi * Wi; ++q) {
    float ws = acc[q * (K + 1) + K];
    float n = 1.0f / (ws > eps ? ws : eps);
    for (int64_t c = 0; c < K; ++c) out[q * K + c] = acc[q * (K + 1) + c] * n;
  }
  free(acc);
}

/* ray_plane_delta + ray_encoding_base (geometry.hpp:343-391) -> [h,w,32]. */
static void ray_encoding_base(const lvsg_camera* input_cam, const lvsg_frustum* fr, int64_t h,
                              int64_t w, float* out) {
  lvsg_camera grid = cam_scaled(input_cam, w, h);
  double ow[3];
  cam_center(&grid, ow);
  const double* tm = fr->camera.cam_from_world;
  double o[3];
  for (int r = 0; r < 3; ++r) {
    double acc = tm[r * 4 + 0] * ow[0];
    acc += tm[r * 4 + 1] * ow[1];
    acc += tm[r * 4 + 2] * ow[2];
    o[r] = acc + tm[r * 4 + 3];
  }
  double inv_span = 1.0 / fr->far_depth - 1.0 / fr->near_depth;
  double half_w = (double)fr->camera.width / 2.0, half_h = (double)fr->camera.height / 2.0;
  for (int64_t i = 0; i < h; ++i)
    for (int64_t j = 0; j < w; ++j) {
      double dw[3], d[3];
      world_dir(&grid, (double)j + 0.5, (double)i + 0.5, dw);
      for (int r = 0; r < 3; ++r) {
        double acc = tm[r * 4 + 0] * dw[0];
        acc += tm[r * 4 + 1] * dw[1];
        acc += tm[r * 4 + 2] * dw[2];
        d[r] = acc;
      }
      double dz = d[2] >= 0 ? fmax(d[2], 1e-6) : fmin(d[2], -1e-6);
      double sx = o[0] - (d[0] / dz) * o[2];
      double sy = o[1] - (d[1] / dz) * o[2];
      double e[2] = {tanh(fr->camera.fx * sx * inv_span / half_w),
                     tanh(fr->camera.fy * sy * inv_span / half_h)};
      float* dst = out + (i * w + j) * 32;
      for (int comp = 0; comp < 2; ++comp)
        for (int oc = 0; oc < 8; ++oc) {
          double arg = ldexp(M_PI, oc) * e[comp];
          dst[comp * 16 + 2 * oc] = (float)sin(arg);
          dst[comp * 16 + 2 * oc + 1] = (float)cos(arg);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* parameters: build_params order (network.hpp:244-317)                      */
/* ------------------------------------------------------------------------ */

enum { TK_BP, TK_U, TK_LC, TK_A, TK_C };
typedef struct {
  int kind, heads;
} token_t;

/* parse_blocks (network.cpp:8-43), assuming a validated config. */
static int parse_blocks(const char* spec, token_t* out, int cap) {
  int n = 0;
  const char* s = spec;
  while (1) {
    const char* e = strchr(s, ',');
    size_t len = e ? (size_t)(e - s) : strlen(s);
    while (len && (*s == ' ' || *s == '\t')) ++s, --len;
    while (len && (s[len - 1] == ' ' || s[len - 1] == '\t')) --len;
    token_t t = {TK_C, 0};
    if (len == 2 && !strncmp(s, "Bp", 2)) t.kind = TK_BP;
    else if (len == 1 && s[0] == 'U') t.kind = TK_U;
    else if (len == 2 && !strncmp(s, "Lc", 2)) t.kind = TK_LC;
    else if (len == 1 && s[0] == 'C') t.kind = TK_C;
    else if (len > 1 && s[0] == 'A') {
      t.kind = TK_A;
      for (size_t i = 1; i < len; ++i) t.heads = t.heads * 10 + (s[i] - '0');
    } else
      return -1;
    if (n < cap) out[n] = t;
    ++n;
    if (!e) break;
    s = e + 1;
  }
  return n;
}

typedef struct {
  const float *w1, *b1, *w2, *b2;
} pair_p;
typedef struct {
  const float *gain, *w1, *b1, *w2, *b2;
} mlp_p;
typedef struct {
  int heads;
  const float** wq;
  const float *wo, *gain;
  int nmlp;
  mlp_p mlp[32];
} fusion_p;
typedef struct {
  int ncol;
  const float *cw1[8], *cb1[8], *cw2[8], *cb2[8];
  const float *stem_w, *stem_b;
  pair_p r1, r2;
  int nfus;
  fusion_p fus[32];
} step_p;
typedef struct {
  const float* init_feature;
  const float *stem_w, *stem_b;
  pair_p lvl_r1[16], lvl_r2[16];
  const float* ray_proj[16];
  const float *w_sigma, *w_depth, *w_appear, *blend_w, *blend_gain;
  step_p steps[LVSG_MAX_STEPS];
} params_t;

static pair_p take_pair(const float** cur, int64_t C) {
  pair_p p;
  p.w1 = *cur, *cur += C * C * 9;
  p.b1 = *cur, *cur += C;
  p.w2 = *cur, *cur += C * C * 9;
  p.b2 = *cur, *cur += C;
  return p;
}

static void bind_params(const lvsg_model_config* cfg, const float* w, params_t* P) {
  const int64_t C = cfg->channels, Ca = cfg->direct_rgb ? 3 : C;
  const float* cur = w;
  memset(P, 0, sizeof(*P));
  P->init_feature = cur, cur += C;
  P->stem_w = cur, cur += C * 27;
  P->stem_b = cur, cur += C;
  for (int64_t k = 0; k < cfg->pyramid_levels; ++k) {
    P->lvl_r1[k] = take_pair(&cur, C);
    P->lvl_r2[k] = take_pair(&cur, C);
    P->ray_proj[k] = cur, cur += 32 * C;
  }
  P->w_sigma = cur, cur += C;
  P->w_depth = cur, cur += C;
  P->w_appear = cur, cur += C * Ca;
  P->blend_w = cur, cur += C * C;
  P->blend_gain = cur, cur += C;
  for (int64_t s = 0; s < cfg->num_steps; ++s) {
    token_t tk[128];
    int n = parse_blocks(cfg->steps[s].blocks, tk, 128);
    step_p* sp = &P->steps[s];
    for (int i = 0; i < n; ++i) {
      if (tk[i].kind == TK_LC) {
        int c = sp->ncol++;
        sp->cw1[c] = cur, cur += 4 * C * C;
        sp->cb1[c] = cur, cur += 2 * C;
        sp->cw2[c] = cur, cur += 2 * C * C;
        sp->cb2[c] = cur, cur += C;
      } else if (tk[i].kind == TK_BP || tk[i].kind == TK_U) {
        int64_t cat = tk[i].kind == TK_U ? 2 * C + Ca + 1 : 2 * C;
        sp->stem_w = cur, cur += C * cat * 9;
        sp->stem_b = cur, cur += C;
        sp->r1 = take_pair(&cur, C);
        sp->r2 = take_pair(&cur, C);
      } else if (tk[i].kind == TK_A) {
        fusion_p* f = &sp->fus[sp->nfus++];
        f->heads = tk[i].heads;
        f->wq = (const float**)malloc(sizeof(float*) * (size_t)f->heads);
        for (int h = 0; h < f->heads; ++h) f->wq[h] = cur, cur += C * C;
        f->wo = cur, cur += f->heads * C * C;
        f->gain = cur, cur += C;
      } else {
        fusion_p* f = &sp->fus[sp->nfus - 1];
        mlp_p* m = &f->mlp[f->nmlp++];
        m->gain = cur, cur += C;
        m->w1 = cur, cur += C * C * 9;
        m->b1 = cur, cur += C;
        m->w2 = cur, cur += C * C * 9;
        m->b2 = cur, cur += C;
      }
    }
  }
}

static void free_params(const lvsg_model_config* cfg, params_t* P) {
  for (int64_t s = 0; s < cfg->num_steps; ++s)
    for (int f = 0; f < P->steps[s].nfus; ++f) free((void*)P->steps[s].fus[f].wq);
}

/* ------------------------------------------------------------------------ */
/* network blocks                                                            */
/* ------------------------------------------------------------------------ */

/* conv_residual on CHW (network.hpp:150-153): x + conv(gelu(conv(x))). */
static void conv_residual(float* x, const pair_p* p, int64_t C, int64_t H, int64_t W, float* t1,
                          float* t2) {
  int64_t n = C * H * W;
  lvso_conv3x3(x, p->w1, p->b1, t1, C, C, H, W);
  for (int64_t i = 0; i < n; ++i) t1[i] = gelu(t1[i]);
  lvso_conv3x3(t1, p->w2, p->b2, t2, C, C, H, W);
  for (int64_t i = 0; i < n; ++i) x[i] = x[i] + t2[i];
}

/* run_update_cnn (network.hpp:155-160): CHW in [Cin,H,W] -> HWC out [H,W,C]. */
static void update_cnn(const float* x_chw, int64_t Cin, const step_p* sp, int64_t C, int64_t H,
                       int64_t W, float* out_hwc) {
  float* h = falloc(C * H * W);
  float* t1 = falloc(C * H * W);
  float* t2 = falloc(C * H * W);
  lvso_conv3x3(x_chw, sp->stem_w, sp->stem_b, h, Cin, C, H, W);
  conv_residual(h, &sp->r1, C, H, W, t1, t2);
  conv_residual(h, &sp->r2, C, H, W, t1, t2);
  chw_to_hwc(h, out_hwc, H, W, C);
  free(h);
  free(t1);
  free(t2);
}

/* decode_linear with K columns (ldm.hpp:58-67). */
static void decode_linear(const float* V, int64_t P, int64_t C, const float* w, int64_t K,
                          float* out) {
  matmul(V, w, out, P, C, K);
}

/* attend_residual + otm_attention (attention.hpp:207-252), in place on V.
 * Texels are processed in chunks; per chunk the per-head query projections
 * s_i = n W_q[i] are one tape.matmul each (k ascending). */
typedef struct {
  const float *D, *s;
  float* cat;
  int64_t C, M, heads, base, cnt;
  float inv_temp, uniform_w;
  int zero;
} attn_ctx;

static void attn_rows(void* p, int64_t b, int64_t e) {
  attn_ctx* a = (attn_ctx*)p;
  const int64_t C = a->C, M = a->M, h = a->heads;
  float logits[1024];
  float w[1024];
  for (int64_t r = b; r < e; ++r) {
    const int64_t q = a->base + r;
    const float* d = a->D + q * M * C;
    float* cat = a->cat + q * h * C;
    for (int64_t i = 0; i < h; ++i) {
      float* head = cat + i * C;
      if (a->zero) {
        for (int64_t m = 0; m < M; ++m) w[m] = a->uniform_w;
      } else {
        const float* sq = a->s + (i * a->cnt + r) * C;
        for (int64_t m = 0; m < M; ++m) logits[m] = dot_blocked(sq, d + m * C, C) * a->inv_temp;
        /* softmax (tape.hpp:390-404): max, exp(x - max), sum ascending, * (1/sum) */
        float mx = logits[0];
        for (int64_t m = 1; m < M; ++m) mx = logits[m] > mx ? logits[m] : mx;
        float sum = 0.f;
        for (int64_t m = 0; m < M; ++m) {
          float ex = expf(logits[m] - mx);
          w[m] = ex;
          sum += ex;
        }
        float inv = 1.0f / sum;
        for (int64_t m = 0; m < M; ++m) w[m] *= inv;
      }
      /* mix_tokens (tape.hpp:542-561) */
      for (int64_t c = 0; c < C; ++c) head[c] = 0.f;
      for (int64_t m = 0; m < M; ++m)
        for (int64_t c = 0; c < C; ++c) head[c] += w[m] * d[m * C + c];
    }
  }
}

static void attend_residual(float* V, const float* D, const fusion_p* f, int64_t P, int64_t C,
                            int64_t M, int zero) {
  const int64_t h = f->heads;
  float* n = falloc(P * C);
  for (int64_t q = 0; q < P; ++q) rms_row(V + q * C, f->gain, n + q * C, C);
  float* cat = falloc(P * h * C);
  const int64_t chunk = 65536;
  float* s = falloc(chunk * h * C);
  attn_ctx a;
  a.D = D;
  a.cat = cat;
  a.s = s;
  a.C = C;
  a.M = M;
  a.heads = h;
  a.inv_temp = (float)(1.0 / sqrt((double)C));
  a.uniform_w = 1.0f / (float)M;
  a.zero = zero;
  for (int64_t b = 0; b < P; b += chunk) {
    int64_t e = b + chunk < P ? b + chunk : P;
    a.base = b;
    a.cnt = e - b;
    if (!zero)
      for (int64_t i = 0; i < h; ++i) matmul(n + b * C, f->wq[i], s + i * (e - b) * C, e - b, C, C);
    par_for(e - b, attn_rows, &a);
  }
  float* o = falloc(P * C);
  matmul(cat, f->wo, o, P, h * C, C);
  for (int64_t i = 0; i < P * C; ++i) V[i] = V[i] + o[i];
  free(n);
  free(cat);
  free(s);
  free(o);
}

/* conv_mlp_residual (attention.hpp:262-267) on V [L,H,W,C]. */
static void conv_mlp(float* V, const mlp_p* m, int64_t L, int64_t H, int64_t W, int64_t C) {
  const int64_t P = H * W;
  float* nrm = falloc(P * C);
  float* x = falloc(C * P);
  float* t1 = falloc(C * P);
  float* t2 = falloc(C * P);
  for (int64_t l = 0; l < L; ++l) {
    float* vl = V + l * P * C;
    for (int64_t q = 0; q < P; ++q) rms_row(vl + q * C, m->gain, nrm + q * C, C);
    hwc_to_chw(nrm, x, H, W, C);
    lvso_conv3x3(x, m->w1, m->b1, t1, C, C, H, W);
    for (int64_t i = 0; i < C * P; ++i) t1[i] = gelu(t1[i]);
    lvso_conv3x3(t1, m->w2, m->b2, t2, C, C, H, W);
    for (int64_t c = 0; c < C; ++c)
      for (int64_t q = 0; q < P; ++q) vl[q * C + c] = vl[q * C + c] + t2[c * P + q];
  }
  free(nrm);
  free(x);
  free(t1);
  free(t2);
}

static void fusion_block(float* V, const float* D, const fusion_p* f, int64_t L, int64_t H,
                         int64_t W, int64_t C, int64_t M, int zero) {
  attend_residual(V, D, f, L * H * W, C, M, zero);
  for (int i = 0; i < f->nmlp; ++i) conv_mlp(V, &f->mlp[i], L, H, W, C);
}

/* layer_collapse (network.hpp:440-455): V [L,H,W,C] -> [L/2,H,W,C]. */
static float* layer_collapse(const float* V, int64_t L, int64_t H, int64_t W, int64_t C,
                             const float* w1, const float* b1, const float* w2, const float* b2) {
  const int64_t P = H * W, L2 = L / 2;
  float* out = falloc(L2 * P * C);
  float* cat = falloc(L2 * P * 2 * C);
  for (int64_t l = 0; l < L2; ++l)
    for (int64_t q = 0; q < P; ++q) {
      const float* a = V + ((2 * l) * P + q) * C;
      const float* b = V + ((2 * l + 1) * P + q) * C;
      float* cq = cat + (l * P + q) * 2 * C;
      for (int64_t c = 0; c < C; ++c) cq[c] = a[c], cq[C + c] = b[c];
    }
  float* h = falloc(L2 * P * 2 * C);
  matmul(cat, w1, h, L2 * P, 2 * C, 2 * C);
  for (int64_t r = 0; r < L2 * P; ++r)
    for (int64_t c = 0; c < 2 * C; ++c) h[r * 2 * C + c] = gelu(h[r * 2 * C + c] + b1[c]);
  float* r = falloc(L2 * P * C);
  matmul(h, w2, r, L2 * P, 2 * C, C);
  for (int64_t l = 0; l < L2; ++l)
    for (int64_t q = 0; q < P; ++q)
      for (int64_t c = 0; c < C; ++c) {
        float a = V[((2 * l) * P + q) * C + c], b = V[((2 * l + 1) * P + q) * C + c];
        float mean = (a + b) * 0.5f;
        float rr = r[(l * P + q) * C + c] + b2[c];
        out[(l * P + q) * C + c] = mean + rr;
      }
  free(cat);
  free(h);
  free(r);
  return out;
}

/* activate_depth over a [L,H,W] logit map (ldm.hpp:73-83). */
static void activate_depth_map(const float* x, float* d, int64_t L, int64_t P, double near,
                               double far) {
  float s1 = (float)(0.5 / (double)L), s2 = (float)(1.0 / near - 1.0 / far),
        s3 = (float)(1.0 / far);
  for (int64_t l = 0; l < L; ++l)
    for (int64_t q = 0; q < P; ++q) d[l * P + q] = depth_act(x[l * P + q], l, L, s1, s2, s3);
}

/* render_to_input_view (ldm.hpp:223-244) -> [Hv,Wv,Ca+1]. */
static int render_to_view(const float* V, int64_t L, int64_t H, int64_t W, int64_t C, int64_t Ca,
                          const params_t* P, const lvsg_frustum* fr, const lvsg_camera* cam,
                          float* out) {
  const int64_t PT = L * H * W, K = Ca + 1;
  float* pre_a = falloc(PT * Ca);
  float* pre_s = falloc(PT);
  float* pre_d = falloc(PT);
  decode_linear(V, PT, C, P->w_appear, Ca, pre_a);
  decode_linear(V, PT, C, P->w_sigma, 1, pre_s);
  decode_linear(V, PT, C, P->w_depth, 1, pre_d);
  float* payload = falloc(PT * K);
  for (int64_t q = 0; q < PT; ++q) {
    for (int64_t c = 0; c < Ca; ++c) payload[q * K + c] = sigmoidf_(pre_a[q * Ca + c]);
    payload[q * K + Ca] = sigmoidf_(pre_s[q]);
  }
  float* depth = falloc(PT);
  activate_depth_map(pre_d, depth, L, H * W, fr->near_depth, fr->far_depth);
  float* pts = falloc(PT * 3);
  int bad = lvso_world_points(fr, depth, L, H, W, pts);
  const int64_t Hv = cam->height, Wv = cam->width, PV = Hv * Wv;
  float* sp = falloc(L * PV * K);
  splat_project(payload, pts, L, H, W, K, cam, sp);
  float* av = falloc(L * PV * Ca);
  float* sv = falloc(L * PV);
  for (int64_t q = 0; q < L * PV; ++q) {
    for (int64_t c = 0; c < Ca; ++c) av[q * Ca + c] = sp[q * K + c];
    sv[q] = sp[q * K + Ca];
  }
  float* color = falloc(PV * Ca);
  over_composite(av, sv, color, L, PV, Ca);
  float* ones = falloc(L * PV);
  for (int64_t q = 0; q < L * PV; ++q) ones[q] = 1.f;
  float* alpha = falloc(PV);
  over_composite(ones, sv, alpha, L, PV, 1);
  for (int64_t q = 0; q < PV; ++q) {
    for (int64_t c = 0; c < Ca; ++c) out[q * K + c] = color[q * Ca + c];
    out[q * K + Ca] = alpha[q];
  }
  free(pre_a);
  free(pre_s);
  free(pre_d);
  free(payload);
  free(depth);
  free(pts);
  free(sp);
  free(av);
  free(sv);
  free(color);
  free(ones);
  free(alpha);
  return bad;
}

/* Stage exports for per-stage parity on oracle-supplied inputs. */
void lvso_attend_residual(float* V, const float* D, int64_t P, int64_t C, int64_t M,
                          int64_t heads, const float* wq, const float* wo, const float* gain,
                          int zero) {
  fusion_p f;
  memset(&f, 0, sizeof(f));
  f.heads = (int)heads;
  f.wq = (const float**)malloc(sizeof(float*) * (size_t)heads);
  for (int64_t h = 0; h < heads; ++h) f.wq[h] = wq + h * C * C;
  f.wo = wo;
  f.gain = gain;
  attend_residual(V, D, &f, P, C, M, zero);
  free((void*)f.wq);
}

int lvso_render_to_view(const lvsg_frustum* fr, const float* V, int64_t L, int64_t H, int64_t W,
                        int64_t C, int64_t Ca, const float* w_appear, const float* w_sigma,
                        const float* w_depth, const lvsg_camera* cam, float* out) {
  params_t P;
  memset(&P, 0, sizeof(P));
  P.w_appear = w_appear;
  P.w_sigma = w_sigma;
  P.w_depth = w_depth;
  return render_to_view(V, L, H, W, C, Ca, &P, fr, cam, out);
}

/* ------------------------------------------------------------------------ */
/* plan (network.cpp:105-151), validated config assumed                      */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t pyr_h[16], pyr_w[16];
  int64_t in_h[LVSG_MAX_STEPS], in_w[LVSG_MAX_STEPS];
  int doubled[LVSG_MAX_STEPS];
  int64_t feat_h[LVSG_MAX_STEPS], feat_w[LVSG_MAX_STEPS], rend_h[LVSG_MAX_STEPS],
      rend_w[LVSG_MAX_STEPS];
  int64_t out_h, out_w;
} plan_t;

static int make_plan(const lvsg_model_config* cfg, int64_t h, int64_t w, plan_t* p, char* err,
                     size_t errlen) {
  for (int64_t k = 0; k < cfg->pyramid_levels; ++k) {
    if (h < 2 || w < 2 || h % 2 || w % 2) {
      snprintf(err, errlen, "plan_forward: pyramid level %lld needs even input dims, got %lldx%lld",
               (long long)k, (long long)h, (long long)w);
      return 1;
    }
    h /= 2;
    w /= 2;
    p->pyr_h[k] = h;
    p->pyr_w[k] = w;
  }
  for (int64_t s = 0; s < cfg->num_steps; ++s) {
    const lvsg_step_config* st = &cfg->steps[s];
    p->in_h[s] = s == 0 ? st->height : cfg->steps[s - 1].height;
    p->in_w[s] = s == 0 ? st->width : cfg->steps[s - 1].width;
    p->doubled[s] = s > 0 && st->height == 2 * p->in_h[s];
    p->feat_h[s] = p->pyr_h[st->pyramid_level];
    p->feat_w[s] = p->pyr_w[st->pyramid_level];
    if (p->doubled[s]) {
      if (st->pyramid_level + 1 >= cfg->pyramid_levels) {
        snprintf(err, errlen, "plan_forward: step %lld doubles resolution but has no coarser level",
                 (long long)s);
        return 1;
      }
      p->rend_h[s] = p->pyr_h[st->pyramid_level + 1];
      p->rend_w[s] = p->pyr_w[st->pyramid_level + 1];
    } else {
      p->rend_h[s] = p->feat_h[s];
      p->rend_w[s] = p->feat_w[s];
    }
  }
  p->out_h = llround((double)cfg->steps[cfg->num_steps - 1].height * cfg->upsample);
  p->out_w = llround((double)cfg->steps[cfg->num_steps - 1].width * cfg->upsample);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* upsample_activate + render_target                                         */
/* ------------------------------------------------------------------------ */

void lvso_upsample_activate(const lvsg_frustum* fr, const float* V, int64_t L, int64_t H, int64_t W,
                            int64_t C, const float* w_depth, const float* w_sigma,
                            const float* logits, int64_t M, int64_t Ho, int64_t Wo, float* depth,
                            float* density, float* blend) {
  const int64_t P = L * H * W, PO = L * Ho * Wo;
  float* xd = falloc(P);
  float* xs = falloc(P);
  decode_linear(V, P, C, w_depth, 1, xd);
  decode_linear(V, P, C, w_sigma, 1, xs);
  float* ud = falloc(PO);
  float* us = falloc(PO);
  resize_planes(xd, ud, L, H, W, Ho, Wo);
  resize_planes(xs, us, L, H, W, Ho, Wo);
  activate_depth_map(ud, depth, L, Ho * Wo, fr->near_depth, fr->far_depth);
  for (int64_t q = 0; q < PO; ++q) density[q] = sigmoidf_(us[q]);
  resize_hwc(logits, blend, L, H, W, M, Ho, Wo);
  for (int64_t q = 0; q < PO; ++q) {
    float* b = blend + q * M;
    float mx = b[0];
    for (int64_t m = 1; m < M; ++m) mx = b[m] > mx ? b[m] : mx;
    float sum = 0.f;
    for (int64_t m = 0; m < M; ++m) {
      float e = expf(b[m] - mx);
      b[m] = e;
      sum += e;
    }
    float inv = 1.0f / sum;
    for (int64_t m = 0; m < M; ++m) b[m] *= inv;
  }
  free(xd);
  free(xs);
  free(ud);
  free(us);
}

/* render_target = world_points + blended_layer_colors + over_composite
 * (ldm.hpp:158-199). */
typedef struct {
  const float *blend, *colors, *mask;
  float* rgb;
  int64_t M;
} blend_ctx;

static void blend_rows(void* p, int64_t b, int64_t e) {
  blend_ctx* c = (blend_ctx*)p;
  const int64_t M = c->M;
  for (int64_t q = b; q < e; ++q) {
    float bm[1024];
    float wsum = 0.f;
    for (int64_t m = 0; m < M; ++m) {
      bm[m] = c->blend[q * M + m] * c->mask[q * M + m];
      wsum += bm[m] * 1.0f;
    }
    float r = 1.0f / (wsum + (float)1e-8);
    float* o = c->rgb + q * 3;
    o[0] = o[1] = o[2] = 0.f;
    for (int64_t m = 0; m < M; ++m) {
      float beta = bm[m] * r;
      const float* col = c->colors + (q * M + m) * 3;
      for (int k = 0; k < 3; ++k) o[k] += beta * col[k];
    }
  }
}

int lvso_render_target(const lvsg_frustum* fr, const float* depth, const float* density,
                       const float* blend, int64_t L, int64_t Ho, int64_t Wo, int64_t M,
                       const float* images, int64_t Hr, int64_t Wr, const lvsg_camera* cams,
                       float* rgb) {
  const int64_t PO = L * Ho * Wo;
  float* pts = falloc(PO * 3);
  int bad = lvso_world_points(fr, depth, L, Ho, Wo, pts);
  float* colors = falloc(PO * M * 3);
  float* mask = falloc(PO * M);
  for (int64_t m = 0; m < M; ++m)
    gather_strided(&cams[m], images + m * Hr * Wr * 3, Hr, Wr, 3, pts, PO, colors + m * 3, M * 3,
                   mask + m, M);
  float* lc = falloc(PO * 3);
  blend_ctx bc = {blend, colors, mask, lc, M};
  par_for(PO, blend_rows, &bc);
  over_composite(lc, density, rgb, L, Ho * Wo, 3);
  free(pts);
  free(colors);
  free(mask);
  free(lc);
  return bad;
}

/* ------------------------------------------------------------------------ */
/* forward (network.hpp:562-603)                                             */
/* ------------------------------------------------------------------------ */

static void seterr(char* err, size_t len, const char* fmt, ...) {
  if (!err || !len) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, len, fmt, ap);
  va_end(ap);
}

int lvso_forward_render(const lvsg_model_config* cfg, int64_t M, const float* enc_images,
                        int64_t He, int64_t We, const lvsg_camera* enc_cams,
                        const float* render_images, int64_t Hr, int64_t Wr,
                        const lvsg_camera* render_cams, const lvsg_frustum* target,
                        const float* weights, float* rgb_out, float* depth_out,
                        float* density_out, float* blend_out, float* logits_out,
                        float* volume_out, char* err, size_t errlen) {
  return lvso_forward_render_ex(cfg, M, enc_images, He, We, enc_cams, render_images, Hr, Wr,
                                render_cams, target, weights, rgb_out, depth_out, density_out,
                                blend_out, logits_out, volume_out, NULL, NULL, err, errlen);
}

int lvso_forward_render_ex(const lvsg_model_config* cfg, int64_t M, const float* enc_images,
                           int64_t He, int64_t We, const lvsg_camera* enc_cams,
                           const float* render_images, int64_t Hr, int64_t Wr,
                           const lvsg_camera* render_cams, const lvsg_frustum* target,
                           const float* weights, float* rgb_out, float* depth_out,
                           float* density_out, float* blend_out, float* logits_out,
                           float* volume_out, float* deltas_out, float* rgb_direct_out, char* err,
                           size_t errlen) {
  if (M != cfg->views) {
    seterr(err, errlen, "forward: expected %lld views", (long long)cfg->views);
    return 1;
  }
  plan_t plan;
  if (make_plan(cfg, He, We, &plan, err, errlen)) return 1;
  const int64_t C = cfg->channels, Ca = cfg->direct_rgb ? 3 : C, K = cfg->pyramid_levels;
  params_t P;
  bind_params(cfg, weights, &P);
  int bad = 0;

  /* --- encode_inputs (network.hpp:368-417) --- */
  float** feats = (float**)calloc((size_t)(M * K), sizeof(float*));
  float** rays = (float**)calloc((size_t)(M * K), sizeof(float*));
  {
    const int64_t hK = He >> K, wK = We >> K;
    for (int64_t m = 0; m < M; ++m) {
      float* chw = falloc(3 * He * We);
      hwc_to_chw(enc_images + m * He * We * 3, chw, He, We, 3);
      int64_t h = He, w = We;
      float* x = falloc(C * h * w);
      lvso_conv3x3(chw, P.stem_w, P.stem_b, x, 3, C, h, w);
      free(chw);
      float* t1 = falloc(C * h * w);
      float* t2 = falloc(C * h * w);
      for (int64_t k = 0; k < K; ++k) {
        conv_residual(x, &P.lvl_r1[k], C, h, w, t1, t2);
        conv_residual(x, &P.lvl_r2[k], C, h, w, t1, t2);
        /* mean_pool2 (tape.hpp:816-836) */
        int64_t ho = h / 2, wo = w / 2;
        float* pooled = falloc(C * ho * wo);
        for (int64_t c = 0; c < C; ++c)
          for (int64_t i = 0; i < ho; ++i)
            for (int64_t j = 0; j < wo; ++j) {
              const float* s = x + c * h * w;
              float sum = s[(2 * i) * w + 2 * j] + s[(2 * i) * w + 2 * j + 1] +
                          s[(2 * i + 1) * w + 2 * j] + s[(2 * i + 1) * w + 2 * j + 1];
              pooled[(c * ho + i) * wo + j] = sum * 0.25f;
            }
        free(x);
        x = pooled;
        h = ho;
        w = wo;
        feats[m * K + k] = falloc(h * w * C);
        chw_to_hwc(x, feats[m * K + k], h, w, C);
      }
      free(x);
      free(t1);
      free(t2);
      if (cfg->ablate_rays) {
        for (int64_t k = 0; k < K; ++k) rays[m * K + k] = falloc(plan.pyr_h[k] * plan.pyr_w[k] * C);
      } else {
        float* base = falloc(hK * wK * 32);
        ray_encoding_base(&enc_cams[m], target, hK, wK, base);
        for (int64_t k = 0; k < K; ++k) {
          int64_t Hk = plan.pyr_h[k], Wk = plan.pyr_w[k];
          float* rb = falloc(Hk * Wk * 32);
          resize_hwc(base, rb, 1, hK, wK, 32, Hk, Wk);
          rays[m * K + k] = falloc(Hk * Wk * C);
          matmul(rb, P.ray_proj[k], rays[m * K + k], Hk * Wk, 32, C);
          free(rb);
        }
        free(base);
      }
    }
  }

  /* --- initialize (network.hpp:459-493) --- */
  int64_t L = cfg->steps[0].layers, H = cfg->steps[0].height, W = cfg->steps[0].width;
  float* V = falloc(L * H * W * C);
  for (int64_t q = 0; q < L * H * W; ++q)
    for (int64_t c = 0; c < C; ++c) V[q * C + c] = 0.f + 1.0f * P.init_feature[c];
  float* deltas = NULL;
  {
    float* depth = falloc(L * H * W);
    double inv_span = 1.0 / target->near_depth - 1.0 / target->far_depth;
    for (int64_t l = 0; l < L; ++l) {
      float anchor = (float)(((double)l + 0.5) / (double)L);
      float d = (float)(1.0 / ((double)anchor * inv_span + 1.0 / target->far_depth));
      for (int64_t q = 0; q < H * W; ++q) depth[l * H * W + q] = d;
    }
    float* pts = falloc(L * H * W * 3);
    bad |= lvso_world_points(target, depth, L, H, W, pts);
    const int64_t lev = cfg->steps[0].pyramid_level, Hf = plan.feat_h[0], Wf = plan.feat_w[0];
    float** upd = (float**)calloc((size_t)M, sizeof(float*));
    lvsg_camera* ucams = (lvsg_camera*)calloc((size_t)M, sizeof(lvsg_camera));
    float* cat = falloc(Hf * Wf * 2 * C);
    float* catc = falloc(Hf * Wf * 2 * C);
    for (int64_t m = 0; m < M; ++m) {
      const float* f = feats[m * K + lev];
      const float* r = rays[m * K + lev];
      for (int64_t q = 0; q < Hf * Wf; ++q)
        for (int64_t c = 0; c < C; ++c) cat[q * 2 * C + c] = f[q * C + c], cat[q * 2 * C + C + c] = r[q * C + c];
      hwc_to_chw(cat, catc, Hf, Wf, 2 * C);
      upd[m] = falloc(Hf * Wf * C);
      update_cnn(catc, 2 * C, &P.steps[0], C, Hf, Wf, upd[m]);
      ucams[m] = cam_scaled(&enc_cams[m], Wf, Hf);
    }
    deltas = falloc(L * H * W * M * C);
    trace_ctx(0, 0, 0, H, W);
    backproject_stack(upd, ucams, M, Hf, Wf, C, pts, L * H * W, deltas);
    for (int64_t m = 0; m < M; ++m) free(upd[m]);
    free(upd);
    free(ucams);
    free(cat);
    free(catc);
    free(depth);
    free(pts);
    for (int f = 0; f < P.steps[0].nfus; ++f)
      fusion_block(V, deltas, &P.steps[0].fus[f], L, H, W, C, M, cfg->ablate_attention);
  }

  /* --- update steps (network.hpp:579-588) --- */
  for (int64_t s = 1; s < cfg->num_steps; ++s) {
    const step_p* sp = &P.steps[s];
    for (int c = 0; c < sp->ncol; ++c) {
      float* nv = layer_collapse(V, L, H, W, C, sp->cw1[c], sp->cb1[c], sp->cw2[c], sp->cb2[c]);
      free(V);
      V = nv;
      L /= 2;
    }
    const int64_t lev = cfg->steps[s].pyramid_level, Hf = plan.feat_h[s], Wf = plan.feat_w[s];
    const int64_t Hn = cfg->steps[s].height, Wn = cfg->steps[s].width;
    const int dbl = plan.doubled[s];
    /* update_block (network.hpp:500-535) */
    float** upd = (float**)calloc((size_t)M, sizeof(float*));
    lvsg_camera* ucams = (lvsg_camera*)calloc((size_t)M, sizeof(lvsg_camera));
    const int64_t Kf = Ca + 1, cin = Kf + 2 * C;
    float* cat = falloc(Hf * Wf * cin);
    float* catc = falloc(Hf * Wf * cin);
    float* fb = falloc(Hf * Wf * Kf);
    for (int64_t m = 0; m < M; ++m) {
      if (cfg->ablate_render) {
        memset(fb, 0, sizeof(float) * (size_t)(Hf * Wf * Kf));
      } else {
        lvsg_camera rcam = cam_scaled(&enc_cams[m], plan.rend_w[s], plan.rend_h[s]);
        float* rv = falloc(plan.rend_h[s] * plan.rend_w[s] * Kf);
        trace_ctx((int)s, 1, (int)m, H, W);
        bad |= render_to_view(V, L, H, W, C, Ca, &P, target, &rcam, rv);
        resize_hwc(rv, fb, 1, plan.rend_h[s], plan.rend_w[s], Kf, Hf, Wf);
        free(rv);
      }
      const float* f = feats[m * K + lev];
      const float* r = rays[m * K + lev];
      for (int64_t q = 0; q < Hf * Wf; ++q) {
        float* dst = cat + q * cin;
        for (int64_t c = 0; c < Kf; ++c) dst[c] = fb[q * Kf + c];
        for (int64_t c = 0; c < C; ++c) dst[Kf + c] = f[q * C + c], dst[Kf + C + c] = r[q * C + c];
      }
      hwc_to_chw(cat, catc, Hf, Wf, cin);
      upd[m] = falloc(Hf * Wf * C);
      update_cnn(catc, cin, sp, C, Hf, Wf, upd[m]);
      ucams[m] = cam_scaled(&enc_cams[m], Wf, Hf);
    }
    free(cat);
    free(catc);
    free(fb);
    float* pre_d = falloc(L * H * W);
    decode_linear(V, L * H * W, C, P.w_depth, 1, pre_d);
    float* d = falloc(L * H * W);
    activate_depth_map(pre_d, d, L, H * W, target->near_depth, target->far_depth);
    float* dd = falloc(L * Hn * Wn);
    resize_planes(d, dd, L, H, W, Hn, Wn);
    float* pts = falloc(L * Hn * Wn * 3);
    bad |= lvso_world_points(target, dd, L, Hn, Wn, pts);
    free(deltas);
    deltas = falloc(L * Hn * Wn * M * C);
    trace_ctx((int)s, 0, 0, Hn, Wn);
    backproject_stack(upd, ucams, M, Hf, Wf, C, pts, L * Hn * Wn, deltas);
    for (int64_t m = 0; m < M; ++m) free(upd[m]);
    free(upd);
    free(ucams);
    free(pre_d);
    free(d);
    free(dd);
    free(pts);
    if (dbl) {
      float* nv = falloc(L * Hn * Wn * C);
      resize_hwc(V, nv, L, H, W, C, Hn, Wn);
      free(V);
      V = nv;
    }
    H = Hn;
    W = Wn;
    for (int f = 0; f < sp->nfus; ++f)
      fusion_block(V, deltas, &sp->fus[f], L, H, W, C, M, cfg->ablate_attention);
  }

  /* --- decode_blend_logits (network.hpp:539-549) --- */
  const int64_t PT = L * H * W;
  float* logits = falloc(PT * M);
  if (!cfg->ablate_attention) {
    float* q = falloc(PT * C);
    for (int64_t i = 0; i < PT; ++i) rms_row(V + i * C, P.blend_gain, q + i * C, C);
    float* qq = falloc(PT * C);
    matmul(q, P.blend_w, qq, PT, C, C);
    float it = (float)(1.0 / sqrt((double)C));
    for (int64_t i = 0; i < PT; ++i)
      for (int64_t m = 0; m < M; ++m)
        logits[i * M + m] = dot_blocked(qq + i * C, deltas + (i * M + m) * C, C) * it;
    free(q);
    free(qq);
  }

  /* --- upsample_activate (ldm.hpp:249-271) --- */
  const int64_t Ho = plan.out_h, Wo = plan.out_w, PO = L * Ho * Wo;
  float* depth = falloc(PO);
  float* density = falloc(PO);
  float* blend = falloc(PO * M);
  lvso_upsample_activate(target, V, L, H, W, C, P.w_depth, P.w_sigma, logits, M, Ho, Wo, depth,
                         density, blend);
  if (depth_out) memcpy(depth_out, depth, sizeof(float) * (size_t)PO);
  if (density_out) memcpy(density_out, density, sizeof(float) * (size_t)PO);
  if (blend_out) memcpy(blend_out, blend, sizeof(float) * (size_t)(PO * M));
  if (logits_out) memcpy(logits_out, logits, sizeof(float) * (size_t)(PT * M));
  if (volume_out) memcpy(volume_out, V, sizeof(float) * (size_t)(PT * C));
  if (deltas_out) memcpy(deltas_out, deltas, sizeof(float) * (size_t)(PT * M * C));
  /* ForwardResult.rgb under direct_rgb (network.hpp:596-601): decode_linear
   * of the appearance head, bilinear resize to the output grid, sigmoid,
   * over-composite with the activated density */
  if (rgb_direct_out && cfg->direct_rgb) {
    float* pa = falloc(PT * 3);
    float* ua = falloc(PO * 3);
    decode_linear(V, PT, C, P.w_appear, 3, pa);
    resize_hwc(pa, ua, L, H, W, 3, Ho, Wo);
    for (int64_t q = 0; q < PO * 3; ++q) ua[q] = sigmoidf_(ua[q]);
    over_composite(ua, density, rgb_direct_out, L, Ho * Wo, 3);
    free(pa);
    free(ua);
  }

  /* --- render_target (ldm.hpp:193-199) --- */
  if (render_images && rgb_out) {
    lvsg_frustum fr = *target;
    bad |= lvso_render_target(&fr, depth, density, blend, L, Ho, Wo, M, render_images, Hr, Wr,
                              render_cams, rgb_out);
  }

  for (int64_t i = 0; i < M * K; ++i) free(feats[i]), free(rays[i]);
  free(feats);
  free(rays);
  free(V);
  free(deltas);
  free(logits);
  free(depth);
  free(density);
  free(blend);
  free_params(cfg, &P);
  if (bad) {
    seterr(err, errlen, "world_points: depth outside the frustum range");
    return 1;
  }
  return 0;
}

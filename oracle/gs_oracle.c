/*
 * gs_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A float64 CPU restatement of the reference hot path (splatlab,
 * /root/reference/pkg/src/splatlab), used as the parity checker for the
 * CUDA library and as the CPU baseline arm of bench.py.  It is never linked
 * into the product; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it (through oracle/oracle.py).
 *
 * Pinned: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py
 * imports splatlab and runs its own project/bin_and_sort/render_forward/
 * render_backward/backward_project/_adam_step on seeded scenes).
 *
 * Structure: per-pixel sequential loops (the brute-force form of the
 * reference's chunked numpy code), tiles in parallel with OpenMP.  All
 * arithmetic is IEEE double without contraction (-ffp-contract=off), in the
 * same operation order as the device geometry chain, so integer outputs
 * (radii, tile rectangles, keys, ranges) are reproducible bit-for-bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16
#define LOWPASS 0.3            /* core.py:13 */
#define GUARD 1.3              /* core.py:16 */
#define SIGMAS 3.0             /* core.py:18 */
#define A_EPS (1.0 / 255.0)    /* rasterizer.py:17 */
#define A_CLAMP 0.99           /* rasterizer.py:18 */
#define SATUR 0.9999           /* rasterizer.py:19 */

typedef struct {
  double R[9], t[3], fx, fy, cx, cy;
  int32_t width, height;
  double near_plane;
} or_camera;

/* sh.py:6-23 */
static const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
static const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                             0.5462742152960396};
static const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                             -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* sh.py:32-63 */
static void basis16(double x, double y, double z, int deg, double b[16]) {
  memset(b, 0, 16 * sizeof(double));
  b[0] = C0;
  if (deg >= 1) { b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x; }
  if (deg >= 2) {
    double xx = x * x, yy = y * y, zz = z * z;
    b[4] = C2[0] * x * y; b[5] = C2[1] * y * z; b[6] = C2[2] * (2.0 * zz - xx - yy);
    b[7] = C2[3] * x * z; b[8] = C2[4] * (xx - yy);
    if (deg >= 3) {
      b[9] = C3[0] * y * (3.0 * xx - yy); b[10] = C3[1] * x * y * z;
      b[11] = C3[2] * y * (4.0 * zz - xx - yy); b[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
      b[13] = C3[4] * x * (4.0 * zz - xx - yy); b[14] = C3[5] * z * (xx - yy);
      b[15] = C3[6] * x * (xx - 3.0 * yy);
    }
  }
}

/* transpose-contracted sh_basis_jacobian (sh.py:66-109): out = sum_k db[k] dB_k/d(dir) */
static void basis16_vjp(double x, double y, double z, int deg, const double db[16], double out[3]) {
  double J[16][3];
  memset(J, 0, sizeof(J));
  if (deg >= 1) { J[1][1] = -C1; J[2][2] = C1; J[3][0] = -C1; }
  if (deg >= 2) {
    J[4][0] = C2[0] * y; J[4][1] = C2[0] * x; J[5][1] = C2[1] * z; J[5][2] = C2[1] * y;
    J[6][0] = C2[2] * (-2.0 * x); J[6][1] = C2[2] * (-2.0 * y); J[6][2] = C2[2] * (4.0 * z);
    J[7][0] = C2[3] * z; J[7][2] = C2[3] * x; J[8][0] = C2[4] * (2.0 * x); J[8][1] = C2[4] * (-2.0 * y);
  }
  if (deg >= 3) {
    double xx = x * x, yy = y * y, zz = z * z;
    J[9][0] = C3[0] * 6.0 * x * y; J[9][1] = C3[0] * (3.0 * xx - 3.0 * yy);
    J[10][0] = C3[1] * y * z; J[10][1] = C3[1] * x * z; J[10][2] = C3[1] * x * y;
    J[11][0] = C3[2] * (-2.0 * x * y); J[11][1] = C3[2] * (4.0 * zz - xx - 3.0 * yy); J[11][2] = C3[2] * 8.0 * y * z;
    J[12][0] = C3[3] * (-6.0 * x * z); J[12][1] = C3[3] * (-6.0 * y * z);
    J[12][2] = C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    J[13][0] = C3[4] * (4.0 * zz - 3.0 * xx - yy); J[13][1] = C3[4] * (-2.0 * x * y); J[13][2] = C3[4] * 8.0 * x * z;
    J[14][0] = C3[5] * 2.0 * x * z; J[14][1] = C3[5] * (-2.0 * y * z); J[14][2] = C3[5] * (xx - yy);
    J[15][0] = C3[6] * (3.0 * xx - 3.0 * yy); J[15][1] = C3[6] * (-6.0 * x * y);
  }
  out[0] = out[1] = out[2] = 0.0;
  for (int k = 0; k < 16; ++k)
    for (int d = 0; d < 3; ++d) out[d] += db[k] * J[k][d];
}

/* quaternion_to_rotation (core.py:170-184) */
static void rot_of(const double q[4], double R[9]) {
  double r = q[0], i = q[1], j = q[2], k = q[3];
  R[0] = 1.0 - 2.0 * (j * j + k * k); R[1] = 2.0 * (i * j - r * k); R[2] = 2.0 * (i * k + r * j);
  R[3] = 2.0 * (i * j + r * k); R[4] = 1.0 - 2.0 * (i * i + k * k); R[5] = 2.0 * (j * k - r * i);
  R[6] = 2.0 * (i * k - r * j); R[7] = 2.0 * (j * k + r * i); R[8] = 1.0 - 2.0 * (i * i + j * j);
}

static void camera_center(const or_camera* c, double out[3]) {
  for (int i = 0; i < 3; ++i) out[i] = -(c->R[i] * c->t[0] + c->R[3 + i] * c->t[1] + c->R[6 + i] * c->t[2]);
}

/* Geometry shared by project and backward_project: view position, J, U=JW,
 * world covariance and its factors.  Returns 0 if culled before the
 * covariance (near / guard band), -1 on zero quaternion, 1 otherwise. */
typedef struct {
  double view[3], u, v, j00, j02, j11, j12, U[6], S[9], M[9], R[9], q[4], qn, s[3];
  double ca, cb, cc, det;
} geom_t;

static int geometry(const double* mean, const double* quat, const double* logs, const or_camera* cam, geom_t* G) {
  for (int i = 0; i < 3; ++i)
    G->view[i] = mean[0] * cam->R[3 * i] + mean[1] * cam->R[3 * i + 1] + mean[2] * cam->R[3 * i + 2] + cam->t[i];
  double x = G->view[0], y = G->view[1], z = G->view[2];
  if (!(z >= cam->near_plane)) return 0;                                 /* core.py:281 */
  G->u = cam->fx * x / z + cam->cx;                                       /* core.py:286-287 */
  G->v = cam->fy * y / z + cam->cy;
  double nx = (G->u - cam->cx) / (0.5 * (double)cam->width);
  double ny = (G->v - cam->cy) / (0.5 * (double)cam->height);
  if (!(fabs(nx) <= GUARD && fabs(ny) <= GUARD)) return 0;                /* core.py:288-293 */
  G->qn = sqrt(quat[0] * quat[0] + quat[1] * quat[1] + quat[2] * quat[2] + quat[3] * quat[3]);
  if (G->qn == 0.0) return -1;                                            /* core.py:164-165 */
  for (int k = 0; k < 4; ++k) G->q[k] = quat[k] / G->qn;
  rot_of(G->q, G->R);
  for (int k = 0; k < 3; ++k) G->s[k] = exp(logs[k]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) G->M[3 * i + j] = G->R[3 * i + j] * G->s[j];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      G->S[3 * i + k] = G->M[3 * i] * G->M[3 * k] + G->M[3 * i + 1] * G->M[3 * k + 1] + G->M[3 * i + 2] * G->M[3 * k + 2];
  double zz = z * z;
  G->j00 = cam->fx / z; G->j02 = -cam->fx * x / zz; G->j11 = cam->fy / z; G->j12 = -cam->fy * y / zz;
  for (int c = 0; c < 3; ++c) {
    G->U[c] = G->j00 * cam->R[c] + G->j02 * cam->R[6 + c];
    G->U[3 + c] = G->j11 * cam->R[3 + c] + G->j12 * cam->R[6 + c];
  }
  double US[6];
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 3; ++k)
      US[3 * r + k] = G->U[3 * r] * G->S[k] + G->U[3 * r + 1] * G->S[3 + k] + G->U[3 * r + 2] * G->S[6 + k];
  G->ca = US[0] * G->U[0] + US[1] * G->U[1] + US[2] * G->U[2] + LOWPASS;  /* core.py:304-307 */
  G->cb = US[0] * G->U[3] + US[1] * G->U[4] + US[2] * G->U[5];
  G->cc = US[3] * G->U[3] + US[4] * G->U[4] + US[5] * G->U[5] + LOWPASS;
  G->det = G->ca * G->cc - G->cb * G->cb;                                 /* core.py:309 */
  return 1;
}

/* project (core.py:266-345) + the tile rectangle of bin_and_sort
 * (rasterizer.py:86-97), N-space outputs; radius 0 = culled.
 * Returns 0, or 2 when a survivor of the near/guard tests had |q| = 0. */
int or_project(int64_t n, const double* means, const double* rots, const double* logs, const double* logits,
               const double* sh, const or_camera* cam, int deg, int32_t* radius, double* mean2d, double* conic,
               double* depth, double* color, int32_t* cmask, double* alpha, int32_t* rect, int64_t* tiles) {
  double C[3];
  camera_center(cam, C);
  int tx = (cam->width + TILE - 1) / TILE, ty = (cam->height + TILE - 1) / TILE;
  int err = 0;
#pragma omp parallel for schedule(static) reduction(| : err)
  for (int64_t g = 0; g < n; ++g) {
    geom_t G;
    radius[g] = 0;
    tiles[g] = 0;
    int st = geometry(means + 3 * g, rots + 4 * g, logs + 3 * g, cam, &G);
    if (st < 0) err |= 2;
    if (st <= 0 || !(G.det > 0.0)) continue;
    double mid = 0.5 * (G.ca + G.cc);                                     /* core.py:317-319 */
    double lam = mid + sqrt(fmax(mid * mid - G.det, 0.0));
    double r = ceil(SIGMAS * sqrt(lam));
    radius[g] = r >= 2147483647.0 ? 2147483647 : (int32_t)r;
    mean2d[2 * g] = G.u;
    mean2d[2 * g + 1] = G.v;
    conic[3 * g] = G.cc / G.det;                                          /* core.py:316 */
    conic[3 * g + 1] = -G.cb / G.det;
    conic[3 * g + 2] = G.ca / G.det;
    depth[g] = G.view[2];
    double x0 = floor((G.u - r) / TILE), x1 = floor((G.u + r) / TILE);
    double y0 = floor((G.v - r) / TILE), y1 = floor((G.v + r) / TILE);
    int valid = (x1 >= 0) && (x0 < tx) && (y1 >= 0) && (y0 < ty);
    int ix0 = (int)fmin(fmax(x0, 0), tx - 1), ix1 = (int)fmin(fmax(x1, 0), tx - 1);
    int iy0 = (int)fmin(fmax(y0, 0), ty - 1), iy1 = (int)fmin(fmax(y1, 0), ty - 1);
    rect[4 * g] = ix0; rect[4 * g + 1] = iy0; rect[4 * g + 2] = ix1; rect[4 * g + 3] = iy1;
    tiles[g] = valid ? (int64_t)(ix1 - ix0 + 1) * (int64_t)(iy1 - iy0 + 1) : 0;
    /* SH colour (core.py:321-326) */
    double d[3] = {means[3 * g] - C[0], means[3 * g + 1] - C[1], means[3 * g + 2] - C[2]};
    double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double b[16];
    basis16(d[0] / dist, d[1] / dist, d[2] / dist, deg, b);
    int m = 0;
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
      for (int k = 0; k < 16; ++k) acc += b[k] * sh[48 * g + 3 * k + c];
      acc += 0.5;
      if (acc > 0.0) m |= 1 << c;
      color[3 * g + c] = acc > 0.0 ? acc : 0.0;
    }
    cmask[g] = m;
    alpha[g] = 1.0 / (1.0 + exp(-logits[g]));                             /* core.py:327 */
  }
  return err;
}

/* ---- binning (rasterizer.py:69-124) ---------------------------------- */
/* The reference expands every splat into its tiles splat-major (row-major
 * tiles inside a splat, rasterizer.py:105-111), packs (tile << 32) | float32
 * depth bits (make_keys, rasterizer.py:55-62) and argsorts stably
 * (rasterizer.py:113-116).  A stable sort on (tile, depth bits) of that
 * expansion orders equal keys by splat index, so the result is the
 * lexicographic (tile, depth bits, index) order.  Restated here in O(N log N
 * + K): the survivors sorted by (depth bits, index), then a stable counting
 * sort by tile (keeps large frames — 10^8 instances — tractable on the host). */
typedef struct {
  uint32_t bits;
  int32_t id;
} dk_t;

static int dk_cmp(const void* a, const void* b) {
  const dk_t* x = (const dk_t*)a;
  const dk_t* y = (const dk_t*)b;
  if (x->bits != y->bits) return x->bits < y->bits ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

int64_t or_bin_count(int64_t n, const int64_t* tiles) {
  int64_t k = 0;
  for (int64_t g = 0; g < n; ++g) k += tiles[g];
  return k;
}

static uint32_t depth_bits(double depth) {
  float f = (float)depth; /* rasterizer.py:61: float32 depth */
  uint32_t bits;
  memcpy(&bits, &f, 4);
  return bits;
}

/* keys (nullable): (tile << 32) | float32(depth) bits per sorted instance;
 * ids: Gaussian index per sorted instance; ranges: [start, end) per tile,
 * empty tiles [0, 0] (rasterizer.py:118-123). */
void or_bin_fill(int64_t n, const int32_t* rect, const int64_t* tiles, const double* depth, int tiles_x,
                 int64_t num_tiles, uint64_t* keys, int32_t* ids, int64_t* ranges) {
  int64_t m = 0;
  for (int64_t g = 0; g < n; ++g) m += tiles[g] != 0;
  dk_t* order = (dk_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(dk_t));
  int64_t* cursor = (int64_t*)calloc((size_t)(num_tiles > 0 ? num_tiles : 1), sizeof(int64_t));
  int64_t o = 0;
  for (int64_t g = 0; g < n; ++g) {
    if (tiles[g] == 0) continue;
    order[o].bits = depth_bits(depth[g]);
    order[o].id = (int32_t)g;
    ++o;
    for (int ty = rect[4 * g + 1]; ty <= rect[4 * g + 3]; ++ty)
      for (int tx = rect[4 * g]; tx <= rect[4 * g + 2]; ++tx) cursor[(int64_t)ty * tiles_x + tx] += 1;
  }
  qsort(order, (size_t)m, sizeof(dk_t), dk_cmp);
  int64_t run = 0;
  for (int64_t t = 0; t < num_tiles; ++t) {
    const int64_t c = cursor[t];
    ranges[2 * t] = c ? run : 0;
    ranges[2 * t + 1] = c ? run + c : 0;
    cursor[t] = run;
    run += c;
  }
  for (int64_t r = 0; r < m; ++r) {
    const int64_t g = order[r].id;
    for (int ty = rect[4 * g + 1]; ty <= rect[4 * g + 3]; ++ty)
      for (int tx = rect[4 * g]; tx <= rect[4 * g + 2]; ++tx) {
        const int64_t t = (int64_t)ty * tiles_x + tx;
        const int64_t pos = cursor[t]++;
        ids[pos] = (int32_t)g;
        if (keys) keys[pos] = ((uint64_t)t << 32) | order[r].bits;
      }
  }
  free(cursor);
  free(order);
}

/* ---- forward blend (rasterizer.py:152-240), one pixel at a time ---------- */
static inline double alpha_at(double px, double py, const double* m2, const double* cn, double al, double* graw,
                              double* araw, double* dxo, double* dyo) {
  double dx = px - m2[0], dy = py - m2[1];
  double power = -0.5 * (cn[0] * dx * dx + cn[2] * dy * dy) - cn[1] * dx * dy;
  double G = power > 0.0 ? 0.0 : exp(power);
  double ar = al * G;
  double a = ar < A_CLAMP ? ar : A_CLAMP;
  if (a < A_EPS) a = 0.0;
  if (graw) *graw = G;
  if (araw) *araw = ar;
  if (dxo) *dxo = dx;
  if (dyo) *dyo = dy;
  return a;
}

void or_render_forward(const double* mean2d, const double* conic, const double* alpha, const double* color,
                       const int32_t* ids, const int64_t* ranges, int width, int height, const double* bg,
                       double* image, double* t_final, int64_t* last) {
  int tx_n = (width + TILE - 1) / TILE, ty_n = (height + TILE - 1) / TILE;
  int64_t ntiles = (int64_t)tx_n * ty_n;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t tile = 0; tile < ntiles; ++tile) {
    int tx = (int)(tile % tx_n), ty = (int)(tile / tx_n);
    int64_t s = ranges[2 * tile], e = ranges[2 * tile + 1];
    for (int row = ty * TILE; row < ty * TILE + TILE && row < height; ++row)
      for (int col = tx * TILE; col < tx * TILE + TILE && col < width; ++col) {
        double px = col + 0.5, py = row + 0.5, T = 1.0, c[3] = {0, 0, 0};
        int64_t lastc = -1;
        for (int64_t i = s; i < e; ++i) {
          int32_t g = ids[i];
          double a = alpha_at(px, py, mean2d + 2 * g, conic + 3 * g, alpha[g], 0, 0, 0, 0);
          if (a == 0.0) continue;
          double tn = T * (1.0 - a);
          if (1.0 - tn > SATUR) break;   /* rasterizer.py:179-180 */
          for (int k = 0; k < 3; ++k) c[k] += T * a * color[3 * g + k];
          T = tn;
          lastc = i;
        }
        int64_t p = (int64_t)row * width + col;
        for (int k = 0; k < 3; ++k) image[3 * p + k] = c[k] + T * bg[k];
        if (t_final) t_final[p] = T;
        if (last) last[p] = lastc;
      }
  }
}

/* ---- backward blend (gradients.py:30-94 via rasterizer.py:253-316) ------
 * grads2d (N,9): d_mean2d x,y | d_conic a,b,c | d_alpha | d_color r,g,b.
 * Walks each tile's list back to front; per splat the pixel contributions
 * are summed locally and added once per tile. */
void or_render_backward(const double* d_image, const double* mean2d, const double* conic, const double* alpha,
                        const double* color, const int32_t* ids, const int64_t* ranges, const double* t_final,
                        const int64_t* last, int width, int height, const double* bg, int64_t n, double* grads2d) {
  int tx_n = (width + TILE - 1) / TILE, ty_n = (height + TILE - 1) / TILE;
  int64_t ntiles = (int64_t)tx_n * ty_n;
  memset(grads2d, 0, (size_t)n * 9 * sizeof(double));
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t tile = 0; tile < ntiles; ++tile) {
    int tx = (int)(tile % tx_n), ty = (int)(tile / tx_n);
    int64_t s = ranges[2 * tile];
    int np = 0, pcol[256], prow[256];
    double T[256], S[256], dl[256][3];
    int64_t lp[256], lmax = -1;
    for (int row = ty * TILE; row < ty * TILE + TILE && row < height; ++row)
      for (int col = tx * TILE; col < tx * TILE + TILE && col < width; ++col) {
        int64_t p = (int64_t)row * width + col;
        pcol[np] = col; prow[np] = row;
        T[np] = t_final[p];
        lp[np] = last[p];
        for (int k = 0; k < 3; ++k) dl[np][k] = d_image[3 * p + k];
        S[np] = (dl[np][0] * bg[0] + dl[np][1] * bg[1] + dl[np][2] * bg[2]) * T[np];  /* gradients.py:78 */
        if (lp[np] > lmax) lmax = lp[np];
        ++np;
      }
    for (int64_t i = lmax; i >= s; --i) {
      int32_t g = ids[i];
      double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      int any = 0;
      for (int q = 0; q < np; ++q) {
        if (i > lp[q]) continue;
        double G, ar, dx, dy;
        double a = alpha_at(pcol[q] + 0.5, prow[q] + 0.5, mean2d + 2 * g, conic + 3 * g, alpha[g], &G, &ar, &dx, &dy);
        if (a == 0.0) continue;
        any = 1;
        T[q] = T[q] / (1.0 - a);              /* transmittance before this splat (gradients.py:69-70) */
        double w = T[q] * a;
        double dc = color[3 * g] * dl[q][0] + color[3 * g + 1] * dl[q][1] + color[3 * g + 2] * dl[q][2];
        double da = T[q] * dc - S[q] / (1.0 - a);   /* gradients.py:81 */
        S[q] += w * dc;
        for (int k = 0; k < 3; ++k) acc[6 + k] += w * dl[q][k];
        if (ar < A_CLAMP) {                   /* gradients.py:83-93 */
          const double* cn = conic + 3 * g;
          double dp = da * ar;
          acc[5] += da * G;
          acc[0] += dp * (cn[0] * dx + cn[1] * dy);
          acc[1] += dp * (cn[1] * dx + cn[2] * dy);
          acc[2] += -0.5 * dp * dx * dx;
          acc[3] += -dp * dx * dy;
          acc[4] += -0.5 * dp * dy * dy;
        }
      }
      if (!any) continue;
      for (int k = 0; k < 9; ++k) {
#pragma omp atomic
        grads2d[9 * (int64_t)g + k] += acc[k];
      }
    }
  }
}

/* ---- backward_project (gradients.py:192-259) + stats (optimizer.py:252-255)
 * out: d_means (N,3), d_rot (N,4), d_logs (N,3), d_logit (N), d_sh (N,48), norm (N). */
void or_backward_project(int64_t n, const double* means, const double* rots, const double* logs,
                         const double* logits, const double* sh, const or_camera* cam, int deg,
                         const int32_t* radius, const int32_t* cmask, const double* grads2d, double* d_means,
                         double* d_rot, double* d_logs, double* d_logit, double* d_sh, double* norm) {
  double C[3];
  camera_center(cam, C);
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < n; ++g) {
    memset(d_means + 3 * g, 0, 3 * sizeof(double));
    memset(d_rot + 4 * g, 0, 4 * sizeof(double));
    memset(d_logs + 3 * g, 0, 3 * sizeof(double));
    memset(d_sh + 48 * g, 0, 48 * sizeof(double));
    d_logit[g] = 0.0;
    norm[g] = 0.0;
    if (radius[g] <= 0) continue;
    const double* g2 = grads2d + 9 * g;
    geom_t G;
    geometry(means + 3 * g, rots + 4 * g, logs + 3 * g, cam, &G);
    double al = 1.0 / (1.0 + exp(-logits[g]));
    d_logit[g] = g2[5] * al * (1.0 - al);                                 /* gradients.py:217 */
    /* conic -> screen covariance: -A Gm A (gradients.py:97-113) */
    double A[4] = {G.cc / G.det, -G.cb / G.det, -G.cb / G.det, G.ca / G.det};
    double Gm[4] = {g2[2], 0.5 * g2[3], 0.5 * g2[3], g2[4]};
    double AG[4], dC[4];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) AG[2 * i + j] = A[2 * i] * Gm[j] + A[2 * i + 1] * Gm[2 + j];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) dC[2 * i + j] = -(AG[2 * i] * A[j] + AG[2 * i + 1] * A[2 + j]);
    /* world covariance: U^T dC U (gradients.py:116-123) */
    double dS[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 2; ++k)
          for (int l = 0; l < 2; ++l) acc += G.U[3 * k + i] * dC[2 * k + l] * G.U[3 * l + j];
        dS[3 * i + j] = acc;
      }
    /* scale and rotation (gradients.py:126-189) */
    double dM[9];
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j) acc += dS[3 * i + j] * G.M[3 * j + k];
        dM[3 * i + k] = 2.0 * acc;
      }
    for (int k = 0; k < 3; ++k) {
      double ds = dM[k] * G.R[k] + dM[3 + k] * G.R[3 + k] + dM[6 + k] * G.R[6 + k];
      d_logs[3 * g + k] = ds * G.s[k];
    }
    /* dR/dq of rot_of, contracted with dR = dM diag(s) */
    double dR[9], dq[4] = {0, 0, 0, 0};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) dR[3 * i + j] = dM[3 * i + j] * G.s[j];
    double r = G.q[0], i_ = G.q[1], j_ = G.q[2], k_ = G.q[3];
    double P[4][9] = {
        {0, -2 * k_, 2 * j_, 2 * k_, 0, -2 * i_, -2 * j_, 2 * i_, 0},
        {0, 2 * j_, 2 * k_, 2 * j_, -4 * i_, -2 * r, 2 * k_, 2 * r, -4 * i_},
        {-4 * j_, 2 * i_, 2 * r, 2 * i_, 0, 2 * k_, -2 * r, 2 * k_, -4 * j_},
        {-4 * k_, -2 * r, 2 * i_, 2 * r, -4 * k_, 2 * j_, 2 * i_, 2 * j_, 0},
    };
    for (int a = 0; a < 4; ++a)
      for (int e = 0; e < 9; ++e) dq[a] += P[a][e] * dR[e];
    double qd = G.q[0] * dq[0] + G.q[1] * dq[1] + G.q[2] * dq[2] + G.q[3] * dq[3];
    for (int a = 0; a < 4; ++a) d_rot[4 * g + a] = (dq[a] - G.q[a] * qd) / G.qn;  /* gradients.py:185 */
    /* view position (gradients.py:236-255) */
    double x = G.view[0], y = G.view[1], z = G.view[2], z2 = z * z, z3 = z2 * z;
    double dt[3] = {G.j00 * g2[0], G.j11 * g2[1], G.j02 * g2[0] + G.j12 * g2[1]};
    double dU[6], dJ[6];
    for (int rr = 0; rr < 2; ++rr)
      for (int l = 0; l < 3; ++l) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) {
          double dcu = dC[2 * rr] * G.U[k] + dC[2 * rr + 1] * G.U[3 + k];
          acc += dcu * G.S[3 * k + l];
        }
        dU[3 * rr + l] = 2.0 * acc;
      }
    for (int rr = 0; rr < 2; ++rr)
      for (int k = 0; k < 3; ++k)
        dJ[3 * rr + k] = dU[3 * rr] * cam->R[3 * k] + dU[3 * rr + 1] * cam->R[3 * k + 1] + dU[3 * rr + 2] * cam->R[3 * k + 2];
    dt[0] += dJ[2] * (-cam->fx / z2);
    dt[1] += dJ[5] * (-cam->fy / z2);
    dt[2] += dJ[0] * (-cam->fx / z2) + dJ[2] * (2.0 * cam->fx * x / z3) + dJ[4] * (-cam->fy / z2) +
             dJ[5] * (2.0 * cam->fy * y / z3);
    /* colour path (gradients.py:219-226) */
    double d[3] = {means[3 * g] - C[0], means[3 * g + 1] - C[1], means[3 * g + 2] - C[2]};
    double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double dir[3] = {d[0] / dist, d[1] / dist, d[2] / dist};
    double b[16], db[16], vj[3];
    basis16(dir[0], dir[1], dir[2], deg, b);
    double dcol[3];
    for (int c = 0; c < 3; ++c) dcol[c] = (cmask[g] >> c) & 1 ? g2[6 + c] : 0.0;
    for (int k = 0; k < 16; ++k) {
      db[k] = 0.0;
      for (int c = 0; c < 3; ++c) {
        d_sh[48 * g + 3 * k + c] = b[k] * dcol[c];
        db[k] += dcol[c] * sh[48 * g + 3 * k + c];
      }
    }
    basis16_vjp(dir[0], dir[1], dir[2], deg, db, vj);
    double dot = dir[0] * vj[0] + dir[1] * vj[1] + dir[2] * vj[2];
    for (int j = 0; j < 3; ++j) {
      double dms = (vj[j] - dir[j] * dot) / dist;
      d_means[3 * g + j] = dt[0] * cam->R[j] + dt[1] * cam->R[3 + j] + dt[2] * cam->R[6 + j] + dms;
    }
    norm[g] = sqrt(g2[0] * g2[0] + g2[1] * g2[1]);                       /* gradients.py:258 */
  }
}

/* Densification statistics over survivors (optimizer.py:252-255). */
void or_stats_update(int64_t n, const int32_t* radius, const double* norm, int height, double* accum_pos_grad,
                     int64_t* accum_count, double* max_radius_frac) {
  for (int64_t g = 0; g < n; ++g) {
    if (radius[g] <= 0) continue;
    accum_pos_grad[g] += norm[g];
    accum_count[g] += 1;
    double f = (double)radius[g] / (double)height;
    if (f > max_radius_frac[g]) max_radius_frac[g] = f;
  }
}

/* Dense Adam on one group (optimizer.py:284-293).  lr_of(e) = lr_head when
 * e % period < head (the SH DC row), else lr. */
void or_adam(int64_t numel, double* p, const double* grad, double* m, double* v, double lr, double lr_head,
             int period, int head, double beta1, double beta2, double eps, int64_t t) {
  double b1 = 1.0 - pow(beta1, (double)t), b2 = 1.0 - pow(beta2, (double)t);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < numel; ++e) {
    double g = grad[e];
    m[e] = m[e] * beta1 + (1.0 - beta1) * g;
    v[e] = v[e] * beta2 + (1.0 - beta2) * g * g;
    double l = (period > 0 && (int)(e % period) < head) ? lr_head : lr;
    p[e] -= l * (m[e] / b1) / (sqrt(v[e] / b2) + eps);
  }
}

/* ---- L1 + D-SSIM loss and image gradient (optimizer.py:141-163; ssim.py:50-84)
 * 11-tap Gaussian window (sigma 1.5), separable, zero padding, per channel.
 * out[0] = loss, out[1] = mean |x-y|, out[2] = mean SSIM; d_image (H,W,3). */
static void filt(const double* in, double* out, double* tmp, int H, int W, const double* w) {
  /* rows then columns; in/out (H,W,3) */
#pragma omp parallel for schedule(static)
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c)
      for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
        for (int k = -5; k <= 5; ++k) {
          int rr = r + k;
          if (rr < 0 || rr >= H) continue;
          acc += w[k + 5] * in[((int64_t)rr * W + c) * 3 + ch];
        }
        tmp[((int64_t)r * W + c) * 3 + ch] = acc;
      }
#pragma omp parallel for schedule(static)
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c)
      for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
        for (int k = -5; k <= 5; ++k) {
          int cc = c + k;
          if (cc < 0 || cc >= W) continue;
          acc += w[k + 5] * tmp[((int64_t)r * W + cc) * 3 + ch];
        }
        out[((int64_t)r * W + c) * 3 + ch] = acc;
      }
}

void or_l1_dssim(const double* x, const double* y, int H, int W, double lambda, double* out, double* d_image) {
  const int64_t n = (int64_t)H * W * 3;
  double w[11], s = 0.0;
  for (int i = 0; i < 11; ++i) { double t = i - 5.0; w[i] = exp(-(t * t) / (2.0 * 1.5 * 1.5)); s += w[i]; }
  for (int i = 0; i < 11; ++i) w[i] /= s;
  double* buf = (double*)malloc(sizeof(double) * (size_t)n * 10);
  double *mx = buf, *my = buf + n, *sxx = buf + 2 * n, *syy = buf + 3 * n, *sxy = buf + 4 * n;
  double *tmp = buf + 5 * n, *prod = buf + 6 * n, *a = buf + 7 * n, *b = buf + 8 * n, *c = buf + 9 * n;
  filt(x, mx, tmp, H, W, w);
  filt(y, my, tmp, H, W, w);
  for (int64_t i = 0; i < n; ++i) prod[i] = x[i] * x[i];
  filt(prod, sxx, tmp, H, W, w);
  for (int64_t i = 0; i < n; ++i) prod[i] = y[i] * y[i];
  filt(prod, syy, tmp, H, W, w);
  for (int64_t i = 0; i < n; ++i) prod[i] = x[i] * y[i];
  filt(prod, sxy, tmp, H, W, w);
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03, d_map = -lambda / (2.0 * (double)n);
  double ssum = 0.0, l1 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double vx = sxx[i] - mx[i] * mx[i], vy = syy[i] - my[i] * my[i], cxy = sxy[i] - mx[i] * my[i];
    double a1 = 2.0 * mx[i] * my[i] + C1, a2 = 2.0 * cxy + C2;
    double b1 = mx[i] * mx[i] + my[i] * my[i] + C1, b2 = vx + vy + C2;
    ssum += (a1 * a2) / (b1 * b2);
    l1 += fabs(x[i] - y[i]);
    /* ssim_backward (ssim.py:67-84) */
    double den = b1 * b2, da1 = d_map * a2 / den, da2 = d_map * a1 / den;
    double db1 = -da1 * (a1 / b1), db2 = -da2 * (a2 / b2);
    a[i] = 2.0 * my[i] * da1 + 2.0 * mx[i] * db1 - 2.0 * my[i] * da2 - 2.0 * mx[i] * db2;
    b[i] = db2;
    c[i] = 2.0 * da2;
  }
  double *fa = mx, *fb = my, *fc = sxx;  /* reuse */
  filt(a, fa, tmp, H, W, w);
  filt(b, fb, tmp, H, W, w);
  filt(c, fc, tmp, H, W, w);
  for (int64_t i = 0; i < n; ++i) {
    double diff = x[i] - y[i];
    double sg = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
    d_image[i] = (1.0 - lambda) * sg / (double)n + fa[i] + 2.0 * x[i] * fb[i] + y[i] * fc[i];
  }
  out[1] = l1 / (double)n;
  out[2] = ssum / (double)n;
  out[0] = (1.0 - lambda) * out[1] + lambda * (1.0 - out[2]) / 2.0;
  free(buf);
}

/* Plain-C restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Parity oracle for the CUDA kernels in paper_1811_05784_b200/csrc.  Every
 * function restates a reference function (file:line under
 * /root/reference/proj) in the same fp64 operation order; compiled with
 * -ffp-contract=off for baseline x86-64 so no FMA is formed.  Arithmetic
 * conventions for the Eigen expressions (dot order etc.) are the ones in
 * oracle/eigen_shim/Eigen/Dense.  Pinned against the reference itself
 * (oracle/_ref, tests/test_oracle_vs_ref.py) and against committed golden
 * fixtures (tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this file's library; the product path never does.
 */
#define _GNU_SOURCE
#include "roomray_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];
const char* ro_last_error(void) { return g_err; }
static void set_err(const char* m) {
  snprintf(g_err, sizeof g_err, "%s", m);
}

/* ------------------------------------------------------------------ vectors
 * Eigen expression order per oracle/eigen_shim/Eigen/Dense. */
typedef struct {
  double x, y, z;
} v3;

static inline v3 mk(double x, double y, double z) {
  v3 r = {x, y, z};
  return r;
}
static inline v3 vadd(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 vsub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 vscale(double s, v3 a) { return mk(s * a.x, s * a.y, s * a.z); }
static inline v3 vdiv(v3 a, double s) { return mk(a.x / s, a.y / s, a.z / s); }
static inline double vdot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static inline v3 vcross(v3 a, v3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double vnorm(v3 a) { return sqrt(vdot(a, a)); }
static inline double comp(v3 a, int k) { return k == 0 ? a.x : (k == 1 ? a.y : a.z); }
/* std::min / std::max semantics */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* ------------------------------------------------------------------ scene */
struct ro_scene {
  int64_t nv, nf;
  int32_t nmat;
  double* verts; /* nv*3 */
  int32_t* tris; /* nf*4 */
  double* alpha; /* nmat*8 */
  double* normals; /* nf*3, face_normal geometry.cpp:9-14 */
  int64_t n_nodes;
  int32_t root, depth;
  int32_t *left, *right, *face;
  double *lo, *hi; /* n_nodes*3 */
};

static inline v3 vert(const ro_scene* s, int i) {
  return mk(s->verts[3 * i], s->verts[3 * i + 1], s->verts[3 * i + 2]);
}

/* TriangleMesh::face_area geometry.cpp:22-26 */
static double face_area(const ro_scene* s, int64_t f) {
  const int32_t* t = s->tris + 4 * f;
  v3 a = vert(s, t[0]);
  v3 e1 = vsub(vert(s, t[1]), a), e2 = vsub(vert(s, t[2]), a);
  return 0.5 * vnorm(vcross(e1, e2));
}

/* geometry.cpp:47-75 */
static int validate_mesh(const ro_scene* s) {
  char buf[256];
  for (int64_t i = 0; i < s->nf; ++i) {
    const int32_t* t = s->tris + 4 * i;
    for (int k = 0; k < 3; ++k)
      if (t[k] < 0 || t[k] >= s->nv) {
        snprintf(buf, sizeof buf, "face %lld references a vertex out of range", (long long)i);
        set_err(buf);
        return 1;
      }
    if (t[3] < 0 || t[3] >= s->nmat) {
      snprintf(buf, sizeof buf, "face %lld references material %d out of range", (long long)i, t[3]);
      set_err(buf);
      return 1;
    }
    if (face_area(s, i) <= 1e-12) {
      snprintf(buf, sizeof buf, "face %lld is degenerate (area <= 1e-12 m^2)", (long long)i);
      set_err(buf);
      return 1;
    }
  }
  for (int32_t m = 0; m < s->nmat; ++m)
    for (int b = 0; b < RO_BANDS; ++b) {
      double a = s->alpha[RO_BANDS * m + b];
      if (a < 0.0 || a > 1.0) {
        set_err("material has absorption outside [0,1]");
        return 1;
      }
    }
  return 0;
}

/* ---------------------------------------------------- tree build
 * Builder::build_range accel_tree.cpp:19-47.  nth_element with the total
 * order (centroid[axis], face) selects a unique lower half, so any selection
 * algorithm yields the reference topology; this one is a quickselect. */
typedef struct {
  const ro_scene* s;
  int32_t* order;
  double* cen; /* nf*3 */
  int64_t count;
} builder;

static inline int key_less(const builder* b, int axis, int32_t fa, int32_t fb) {
  double ca = b->cen[3 * fa + axis], cb = b->cen[3 * fb + axis];
  if (ca != cb) return ca < cb;
  return fa < fb;
}

static void select_nth(builder* b, int axis, int64_t lo, int64_t hi, int64_t nth) {
  int32_t* a = b->order;
  while (hi - lo > 1) {
    int64_t mid = lo + (hi - lo) / 2, pi;
    int32_t x = a[lo], y = a[mid], z = a[hi - 1];
    if (key_less(b, axis, x, y))
      pi = key_less(b, axis, y, z) ? mid : (key_less(b, axis, x, z) ? hi - 1 : lo);
    else
      pi = key_less(b, axis, x, z) ? lo : (key_less(b, axis, y, z) ? hi - 1 : mid);
    int32_t t = a[pi];
    a[pi] = a[hi - 1];
    a[hi - 1] = t;
    const int32_t p = a[hi - 1];
    int64_t store = lo;
    for (int64_t i = lo; i < hi - 1; ++i)
      if (key_less(b, axis, a[i], p)) {
        t = a[i];
        a[i] = a[store];
        a[store] = t;
        ++store;
      }
    a[hi - 1] = a[store];
    a[store] = p;
    if (nth == store) return;
    if (nth < store)
      hi = store;
    else
      lo = store + 1;
  }
}

static int32_t build_range(builder* b, int64_t begin, int64_t end) {
  const ro_scene* s = b->s;
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX};
  double hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  for (int64_t i = begin; i < end; ++i) {
    const int32_t* t = s->tris + 4 * b->order[i];
    for (int v = 0; v < 3; ++v)
      for (int k = 0; k < 3; ++k) {
        double c = s->verts[3 * t[v] + k];
        lo[k] = smin(lo[k], c);
        hi[k] = smax(hi[k], c);
      }
  }
  int32_t left = -1, right = -1, face = -1;
  if (end - begin == 1) {
    face = b->order[begin];
  } else {
    double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    int axis = 0;
    for (int k = 1; k < 3; ++k)
      if (ext[k] > ext[axis]) axis = k; /* first index on ties */
    int64_t mid = begin + (end - begin) / 2;
    select_nth(b, axis, begin, end, mid);
    /* after selection [begin,mid) holds the (mid-begin) smallest keys */
    left = build_range(b, begin, mid);
    right = build_range(b, mid, end);
  }
  int64_t id = b->count++;
  ro_scene* ms = (ro_scene*)s;
  ms->left[id] = left;
  ms->right[id] = right;
  ms->face[id] = face;
  for (int k = 0; k < 3; ++k) {
    ms->lo[3 * id + k] = lo[k];
    ms->hi[3 * id + k] = hi[k];
  }
  return (int32_t)id;
}

static int depth_below(const ro_scene* s, int32_t i) {
  if (s->face[i] >= 0) return 0;
  int a = depth_below(s, s->left[i]), c = depth_below(s, s->right[i]);
  return 1 + (a > c ? a : c);
}

ro_scene* ro_scene_create(const double* verts, int64_t nv, const int32_t* tris,
                          int64_t nf, const double* alpha, int32_t nmat,
                          int validate) {
  if (nf <= 0) {
    set_err("cannot build a tree over an empty mesh");
    return NULL;
  }
  ro_scene* s = (ro_scene*)calloc(1, sizeof(ro_scene));
  s->nv = nv;
  s->nf = nf;
  s->nmat = nmat;
  s->verts = (double*)malloc(sizeof(double) * 3 * (nv > 0 ? nv : 1));
  s->tris = (int32_t*)malloc(sizeof(int32_t) * 4 * nf);
  s->alpha = (double*)malloc(sizeof(double) * RO_BANDS * (nmat > 0 ? nmat : 1));
  memcpy(s->verts, verts, sizeof(double) * 3 * nv);
  memcpy(s->tris, tris, sizeof(int32_t) * 4 * nf);
  if (nmat > 0) memcpy(s->alpha, alpha, sizeof(double) * RO_BANDS * nmat);
  if (validate && validate_mesh(s)) {
    ro_scene_destroy(s);
    return NULL;
  }
  s->normals = (double*)malloc(sizeof(double) * 3 * nf);
  for (int64_t f = 0; f < nf; ++f) {
    const int32_t* t = s->tris + 4 * f;
    v3 a = vert(s, t[0]);
    v3 n = vcross(vsub(vert(s, t[1]), a), vsub(vert(s, t[2]), a));
    double z = vdot(n, n);
    if (z > 0.0) n = vdiv(n, sqrt(z)); /* normalized() */
    s->normals[3 * f] = n.x;
    s->normals[3 * f + 1] = n.y;
    s->normals[3 * f + 2] = n.z;
  }
  s->n_nodes = 2 * nf - 1;
  s->left = (int32_t*)malloc(sizeof(int32_t) * s->n_nodes);
  s->right = (int32_t*)malloc(sizeof(int32_t) * s->n_nodes);
  s->face = (int32_t*)malloc(sizeof(int32_t) * s->n_nodes);
  s->lo = (double*)malloc(sizeof(double) * 3 * s->n_nodes);
  s->hi = (double*)malloc(sizeof(double) * 3 * s->n_nodes);
  builder b;
  b.s = s;
  b.count = 0;
  b.order = (int32_t*)malloc(sizeof(int32_t) * nf);
  b.cen = (double*)malloc(sizeof(double) * 3 * nf);
  for (int64_t f = 0; f < nf; ++f) {
    b.order[f] = (int32_t)f;
    const int32_t* t = s->tris + 4 * f;
    v3 c = vdiv(vadd(vadd(vert(s, t[0]), vert(s, t[1])), vert(s, t[2])), 3.0);
    b.cen[3 * f] = c.x;
    b.cen[3 * f + 1] = c.y;
    b.cen[3 * f + 2] = c.z;
  }
  s->root = build_range(&b, 0, nf);
  s->depth = depth_below(s, s->root);
  free(b.order);
  free(b.cen);
  return s;
}

void ro_scene_destroy(ro_scene* s) {
  if (!s) return;
  free(s->verts);
  free(s->tris);
  free(s->alpha);
  free(s->normals);
  free(s->left);
  free(s->right);
  free(s->face);
  free(s->lo);
  free(s->hi);
  free(s);
}

int64_t ro_tree_size(const ro_scene* s, int32_t* root, int32_t* depth) {
  *root = s->root;
  *depth = s->depth;
  return s->n_nodes;
}

void ro_tree_nodes(const ro_scene* s, int32_t* left, int32_t* right,
                   int32_t* face, double* lo, double* hi) {
  memcpy(left, s->left, sizeof(int32_t) * s->n_nodes);
  memcpy(right, s->right, sizeof(int32_t) * s->n_nodes);
  memcpy(face, s->face, sizeof(int32_t) * s->n_nodes);
  memcpy(lo, s->lo, sizeof(double) * 3 * s->n_nodes);
  memcpy(hi, s->hi, sizeof(double) * 3 * s->n_nodes);
}

void ro_face_normals(const ro_scene* s, double* normals) {
  memcpy(normals, s->normals, sizeof(double) * 3 * s->nf);
}

/* TriangleMesh::bounds geometry.cpp:41-45 */
void ro_scene_bounds(const ro_scene* s, double* lo, double* hi) {
  for (int k = 0; k < 3; ++k) {
    lo[k] = DBL_MAX;
    hi[k] = -DBL_MAX;
  }
  for (int64_t i = 0; i < s->nv; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = smin(lo[k], s->verts[3 * i + k]);
      hi[k] = smax(hi[k], s->verts[3 * i + k]);
    }
}

/* ---------------------------------------------------- queries */
typedef struct {
  int ok;
  double delta;
  v3 point;
  int32_t face;
} hit_t;

/* intersect_triangle geometry.cpp:77-106 (Moller-Trumbore, double-sided) */
static inline hit_t intersect_triangle(const ro_scene* s, v3 o, v3 d, int32_t f) {
  hit_t h;
  h.ok = 0;
  const int32_t* t = s->tris + 4 * f;
  v3 va = vert(s, t[0]);
  v3 e1 = vsub(vert(s, t[1]), va);
  v3 e2 = vsub(vert(s, t[2]), va);
  v3 p = vcross(d, e2);
  double det = vdot(e1, p);
  if (det == 0.0) return h;
  double inv = 1.0 / det;
  v3 tv = vsub(o, va);
  double lambda = vdot(tv, p) * inv;
  if (lambda < 0.0 || lambda > 1.0) return h;
  v3 q = vcross(tv, e1);
  double mu = vdot(d, q) * inv;
  if (mu < 0.0 || lambda + mu > 1.0) return h;
  double delta = vdot(e2, q) * inv;
  if (delta <= 1e-6) return h; /* kSelfHitEpsilon types.hpp:31 */
  h.ok = 1;
  h.delta = delta;
  h.point = vadd(o, vscale(delta, d));
  h.face = f;
  return h;
}

/* graze_margin accel_tree.cpp:93 */
static inline double graze(double t) { return 1e-12 * smax(1.0, fabs(t)); }

/* ray_box_entry accel_tree.cpp:97-119 */
static inline int box_entry(const ro_scene* s, int32_t node, v3 o, v3 d, double* out) {
  double t_near = 0.0, t_far = INFINITY;
  const double* lo = s->lo + 3 * node;
  const double* hi = s->hi + 3 * node;
  for (int k = 0; k < 3; ++k) {
    double ok = comp(o, k), dk = comp(d, k);
    if (dk == 0.0) {
      double m = graze(ok);
      if (ok < lo[k] - m || ok > hi[k] + m) return 0;
      continue;
    }
    double inv = 1.0 / dk;
    double ta = (lo[k] - ok) * inv;
    double tb = (hi[k] - ok) * inv;
    if (ta > tb) {
      double t = ta;
      ta = tb;
      tb = t;
    }
    t_near = smax(t_near, ta);
    t_far = smin(t_far, tb);
  }
  if (t_near > t_far + graze(t_far)) return 0;
  *out = t_near;
  return 1;
}

/* nearest_hit accel_tree.cpp:125-181, with optional visit counters */
static hit_t nearest_hit(const ro_scene* s, v3 o, v3 d, int32_t* n_int, int32_t* n_leaf) {
  hit_t best;
  best.ok = 0;
  int32_t ci = 0, cl = 0;
  struct {
    int32_t node;
    double t;
  } stack[64];
  int top = 0;
  double t0;
  if (s->root >= 0 && box_entry(s, s->root, o, d, &t0)) {
    stack[top].node = s->root;
    stack[top].t = t0;
    ++top;
  }
  while (top > 0) {
    --top;
    int32_t node = stack[top].node;
    double te = stack[top].t;
    if (best.ok && te > best.delta + graze(best.delta)) continue;
    if (s->face[node] >= 0) {
      ++cl;
      hit_t h = intersect_triangle(s, o, d, s->face[node]);
      if (h.ok && (!best.ok || h.delta < best.delta ||
                   (h.delta == best.delta && h.face < best.face)))
        best = h;
      continue;
    }
    ++ci;
    double tl = 0, tr = 0;
    int hl = box_entry(s, s->left[node], o, d, &tl);
    int hr = box_entry(s, s->right[node], o, d, &tr);
    int32_t nn = s->left[node], fn = s->right[node];
    int hn = hl, hf = hr;
    double tn = tl, tf = tr;
    if ((hn && hf && tf < tn) || !hn) {
      int32_t xi = nn;
      nn = fn;
      fn = xi;
      int xh = hn;
      hn = hf;
      hf = xh;
      double xt = tn;
      tn = tf;
      tf = xt;
    }
    if (hf && (!best.ok || tf <= best.delta + graze(best.delta))) {
      stack[top].node = fn;
      stack[top].t = tf;
      ++top;
    }
    if (hn && (!best.ok || tn <= best.delta + graze(best.delta))) {
      stack[top].node = nn;
      stack[top].t = tn;
      ++top;
    }
  }
  if (n_int) *n_int = ci;
  if (n_leaf) *n_leaf = cl;
  return best;
}

/* nearest_hit_brute accel_tree.cpp:183-191 */
static hit_t nearest_hit_brute(const ro_scene* s, v3 o, v3 d) {
  hit_t best;
  best.ok = 0;
  for (int64_t f = 0; f < s->nf; ++f) {
    hit_t h = intersect_triangle(s, o, d, (int32_t)f);
    if (h.ok && (!best.ok || h.delta < best.delta)) best = h;
  }
  return best;
}

int ro_nearest_hit(const ro_scene* s, const double* o, const double* d,
                   int64_t n, int brute, int32_t* face, double* delta,
                   double* point, int32_t* n_int, int32_t* n_leaf) {
  for (int64_t i = 0; i < n; ++i) {
    v3 org = mk(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
    v3 dir = mk(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
    int32_t ci = 0, cl = 0;
    hit_t h = brute ? nearest_hit_brute(s, org, dir) : nearest_hit(s, org, dir, &ci, &cl);
    face[i] = h.ok ? h.face : -1;
    delta[i] = h.ok ? h.delta : 0.0;
    point[3 * i] = h.ok ? h.point.x : 0.0;
    point[3 * i + 1] = h.ok ? h.point.y : 0.0;
    point[3 * i + 2] = h.ok ? h.point.z : 0.0;
    if (n_int) n_int[i] = ci;
    if (n_leaf) n_leaf[i] = cl;
  }
  return 0;
}

/* intersect_sphere geometry.cpp:115-128 */
static inline int sphere(v3 o, v3 d, v3 c, double r, double* out) {
  v3 oc = vsub(o, c);
  double b = vdot(d, oc);
  double cc = vdot(oc, oc) - r * r;
  double disc = b * b - cc;
  if (disc < 0.0) return 0;
  double sq = sqrt(disc);
  double nr = -b - sq;
  if (nr > 0.0) {
    *out = nr;
    return 1;
  }
  double fr = -b + sq;
  if (fr > 0.0) {
    *out = fr;
    return 1;
  }
  return 0;
}

int ro_intersect_sphere(const double* o, const double* d, const double* c,
                        double r, double* out) {
  return sphere(mk(o[0], o[1], o[2]), mk(d[0], d[1], d[2]), mk(c[0], c[1], c[2]), r, out);
}

/* fibonacci_directions emission.cpp:17-29.  The reference's
 * rho*std::cos(phi), rho*std::sin(phi) compiles (g++ -O2, objdump of
 * oracle/_ref/obj/emission.o) to ONE glibc sincos() call, whose results can
 * differ from separate sin()/cos() calls, so the restatement calls sincos
 * explicitly rather than relying on gcc to merge the pair. */
static inline v3 fib_dir(int64_t k, int64_t n) {
  const double golden = (1.0 + sqrt(5.0)) / 2.0;
  const double step = 2.0 * M_PI * (1.0 - 1.0 / golden);
  double z = 1.0 - (2.0 * (double)k + 1.0) / (double)n;
  double rho = sqrt(smax(0.0, 1.0 - z * z));
  double phi = step * (double)k;
  double s, c;
  sincos(phi, &s, &c);
  return mk(rho * c, rho * s, z);
}

void ro_fibonacci(int64_t n, int64_t first, int64_t stride, int64_t count, double* out) {
  if (stride <= 0) {
    first = 0;
    stride = 1;
    count = n;
  }
  for (int64_t i = 0; i < count; ++i) {
    v3 v = fib_dir(first + i * stride, n);
    out[3 * i] = v.x;
    out[3 * i + 1] = v.y;
    out[3 * i + 2] = v.z;
  }
}

/* ---------------------------------------------------- trace */
typedef struct {
  int32_t recv, ray, step;
  double point[3], dir[3], path;
  double mult[RO_BANDS];
  int64_t hist_off; /* into the owning buffer's hist array */
  int32_t hist_len;
} cap_t;

typedef struct {
  cap_t* caps;
  int64_t n, cap;
  int32_t* hist;
  int64_t nh, caph;
} capbuf;

static void cb_push(capbuf* b, const cap_t* c, const int32_t* h, int32_t len) {
  if (b->n == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 1024;
    b->caps = (cap_t*)realloc(b->caps, sizeof(cap_t) * b->cap);
  }
  if (b->nh + len > b->caph) {
    while (b->nh + len > b->caph) b->caph = b->caph ? 2 * b->caph : 4096;
    b->hist = (int32_t*)realloc(b->hist, sizeof(int32_t) * b->caph);
  }
  b->caps[b->n] = *c;
  b->caps[b->n].hist_off = b->nh;
  b->caps[b->n].hist_len = len;
  if (len) memcpy(b->hist + b->nh, h, sizeof(int32_t) * len);
  b->nh += len;
  b->n++;
}

struct ro_trace {
  int32_t iterations, truncated;
  int64_t escaped, out_of_range, ray_bounces, sum_int, sum_leaf;
  double max_range;
  capbuf all;
};

typedef struct {
  const ro_scene* s;
  v3 src;
  int64_t n;
  const double* rc;
  const double* rr;
  const double* rng; /* capture range per receiver */
  const double* dirs; /* optional caller directions (count x 3), else the lattice */
  int32_t n_recv;
  int32_t max_it;
  double max_range; /* kill range: the largest of rng */
  int64_t first, stride, begin, end;
  /* outputs */
  capbuf buf;
  int32_t max_steps;
  int64_t escaped, oor, alive, bounces, sum_int, sum_leaf;
} worker;

/* step_ray tracer.cpp:19-62, applied to one ray until it dies or the
 * iteration cap (tracer.cpp:124-132): rays are independent, so running each
 * ray to completion yields the same captures as the iteration-synchronous
 * loop once both are sorted by (ray, path) (tracer.cpp:143-147). */
static void* trace_worker(void* arg) {
  worker* w = (worker*)arg;
  const ro_scene* s = w->s;
  int32_t* hist = (int32_t*)malloc(sizeof(int32_t) * (w->max_it > 0 ? w->max_it : 1));
  for (int64_t i = w->begin; i < w->end; ++i) {
    int64_t k = w->first + i * w->stride;
    v3 o = w->src;
    v3 d = w->dirs ? mk(w->dirs[3 * i], w->dirs[3 * i + 1], w->dirs[3 * i + 2]) : fib_dir(k, w->n);
    double path = 0.0;
    double mult[RO_BANDS];
    for (int b = 0; b < RO_BANDS; ++b) mult[b] = 1.0;
    int alive = 1, steps = 0, len = 0;
    while (alive && steps < w->max_it) {
      ++steps;
      int32_t ci = 0, cl = 0;
      hit_t wall = nearest_hit(s, o, d, &ci, &cl);
      w->sum_int += ci;
      w->sum_leaf += cl;
      for (int32_t r = 0; r < w->n_recv; ++r) {
        double sd;
        v3 c = mk(w->rc[3 * r], w->rc[3 * r + 1], w->rc[3 * r + 2]);
        if (sphere(o, d, c, w->rr[r], &sd) && (!wall.ok || sd < wall.delta)) {
          double L = path + sd;
          if (L <= w->rng[r]) {
            cap_t cp;
            cp.recv = r;
            cp.ray = (int32_t)k;
            cp.step = steps;
            v3 p = vadd(o, vscale(sd, d));
            cp.point[0] = p.x;
            cp.point[1] = p.y;
            cp.point[2] = p.z;
            cp.dir[0] = d.x;
            cp.dir[1] = d.y;
            cp.dir[2] = d.z;
            cp.path = L;
            memcpy(cp.mult, mult, sizeof mult);
            cb_push(&w->buf, &cp, hist, len);
          }
        }
      }
      if (!wall.ok) {
        alive = 0;
        break;
      }
      const double* nn = s->normals + 3 * wall.face;
      v3 n = mk(nn[0], nn[1], nn[2]);
      if (vdot(n, d) > 0.0) n = mk(-n.x, -n.y, -n.z);
      o = wall.point;
      double sdot = 2.0 * vdot(d, n);
      d = vsub(d, vscale(sdot, n)); /* reflect tracer.hpp:33-37 */
      path += wall.delta;
      const double* al = s->alpha + RO_BANDS * s->tris[4 * wall.face + 3];
      for (int b = 0; b < RO_BANDS; ++b) mult[b] *= (1.0 - al[b]);
      hist[len++] = wall.face;
      if (path > w->max_range) alive = 0;
    }
    w->bounces += steps;
    if (steps > w->max_steps) w->max_steps = steps;
    if (alive)
      w->alive++;
    else if (path > w->max_range)
      w->oor++;
    else
      w->escaped++;
  }
  free(hist);
  return NULL;
}

static int cap_cmp(const void* a, const void* b) {
  const cap_t* x = (const cap_t*)a;
  const cap_t* y = (const cap_t*)b;
  if (x->recv != y->recv) return x->recv < y->recv ? -1 : 1;
  if (x->ray != y->ray) return x->ray < y->ray ? -1 : 1;
  if (x->step != y->step) return x->step < y->step ? -1 : 1;
  return 0;
}

ro_trace* ro_trace_run(const ro_scene* s, const double* src, int64_t ray_count,
                       const double* recv_centers, const double* recv_radii,
                       int32_t n_recv, int32_t max_iterations, double max_range,
                       int32_t threads, int64_t first, int64_t stride,
                       int64_t count) {
  return ro_trace_run_dirs(s, src, ray_count, recv_centers, recv_radii, n_recv, max_iterations, max_range,
                           threads, first, stride, count, NULL);
}

/* Several receivers on one set of trajectories (a receiver never alters a
 * ray, tracer.cpp:27-29): receiver r captures while L <= its own
 * resolved_max_range (tracer.cpp:10-15), rays die past the largest, which
 * reproduces one reference trace() per receiver.  dirs (count x 3, may be
 * NULL) replaces the lattice directions of the traced rays (the Ray span of
 * step(), tracer.hpp:43). */
ro_trace* ro_trace_run_dirs(const ro_scene* s, const double* src, int64_t ray_count,
                            const double* recv_centers, const double* recv_radii,
                            int32_t n_recv, int32_t max_iterations, double max_range,
                            int32_t threads, int64_t first, int64_t stride,
                            int64_t count, const double* dirs) {
  for (int32_t r = 0; r < n_recv; ++r)
    if (recv_radii[r] <= 0.0) {
      set_err("receiver radius must be > 0");
      return NULL;
    }
  if (n_recv < 1 || n_recv > 64) {
    set_err("n_recv must be in [1, 64]");
    return NULL;
  }
  if (ray_count < 1) {
    set_err("source ray_count must be >= 1");
    return NULL;
  }
  if (stride <= 0) {
    first = 0;
    stride = 1;
    count = ray_count;
  }
  if (count <= 0 || first + (count - 1) * stride >= ray_count)
    count = (ray_count - first + stride - 1) / stride;
  /* resolved_max_range tracer.cpp:10-15, per receiver */
  double rng[64];
  double mr = 0.0;
  for (int32_t r = 0; r < n_recv; ++r) {
    rng[r] = max_range > 0.0 ? max_range : 0.5 * recv_radii[r] * sqrt((double)ray_count);
    if (rng[r] > mr) mr = rng[r];
  }
  if (threads < 1) threads = 1;
  if (count < threads) threads = count > 0 ? (int32_t)count : 1;
  worker* ws = (worker*)calloc(threads, sizeof(worker));
  pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
  int64_t chunk = (count + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    worker* w = ws + t;
    w->s = s;
    w->src = mk(src[0], src[1], src[2]);
    w->n = ray_count;
    w->rc = recv_centers;
    w->rr = recv_radii;
    w->rng = rng;
    w->dirs = dirs;
    w->n_recv = n_recv;
    w->max_it = max_iterations;
    w->max_range = mr;
    w->first = first;
    w->stride = stride;
    w->begin = t * chunk;
    w->end = (t + 1) * chunk < count ? (t + 1) * chunk : count;
    if (w->begin > w->end) w->begin = w->end;
    if (threads == 1)
      trace_worker(w);
    else
      pthread_create(th + t, NULL, trace_worker, w);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  ro_trace* r = (ro_trace*)calloc(1, sizeof(ro_trace));
  r->max_range = mr;
  int64_t alive = 0;
  int32_t max_steps = 0;
  for (int t = 0; t < threads; ++t) {
    worker* w = ws + t;
    r->escaped += w->escaped;
    r->out_of_range += w->oor;
    r->ray_bounces += w->bounces;
    r->sum_int += w->sum_int;
    r->sum_leaf += w->sum_leaf;
    alive += w->alive;
    if (w->max_steps > max_steps) max_steps = w->max_steps;
    for (int64_t i = 0; i < w->buf.n; ++i) {
      cap_t* c = w->buf.caps + i;
      cb_push(&r->all, c, w->buf.hist + c->hist_off, c->hist_len);
    }
    free(w->buf.caps);
    free(w->buf.hist);
  }
  r->iterations = max_iterations > 0 ? max_steps : 0;
  r->truncated = alive > 0;
  if (r->all.n > 1) qsort(r->all.caps, r->all.n, sizeof(cap_t), cap_cmp);
  free(ws);
  free(th);
  return r;
}

void ro_trace_info(const ro_trace* t, int32_t* iterations, int32_t* truncated,
                   int64_t* escaped, int64_t* out_of_range, double* max_range,
                   int64_t* n_captures, int64_t* total_hist,
                   int64_t* ray_bounces, int64_t* sum_n_int,
                   int64_t* sum_n_leaf) {
  *iterations = t->iterations;
  *truncated = t->truncated;
  *escaped = t->escaped;
  *out_of_range = t->out_of_range;
  *max_range = t->max_range;
  *n_captures = t->all.n;
  *total_hist = t->all.nh;
  *ray_bounces = t->ray_bounces;
  *sum_n_int = t->sum_int;
  *sum_n_leaf = t->sum_leaf;
}

void ro_trace_captures(const ro_trace* t, int32_t* recv, int32_t* ray,
                       double* point, double* dir, double* path, double* mult,
                       int64_t* hist_off, int32_t* hist) {
  int64_t off = 0;
  for (int64_t i = 0; i < t->all.n; ++i) {
    const cap_t* c = t->all.caps + i;
    if (recv) recv[i] = c->recv;
    ray[i] = c->ray;
    for (int k = 0; k < 3; ++k) {
      point[3 * i + k] = c->point[k];
      dir[3 * i + k] = c->dir[k];
    }
    path[i] = c->path;
    for (int b = 0; b < RO_BANDS; ++b) mult[RO_BANDS * i + b] = c->mult[b];
    hist_off[i] = off;
    memcpy(hist + off, t->all.hist + c->hist_off, sizeof(int32_t) * c->hist_len);
    off += c->hist_len;
  }
  hist_off[t->all.n] = off;
}

void ro_trace_free(ro_trace* t) {
  if (!t) return;
  free(t->all.caps);
  free(t->all.hist);
  free(t);
}

/* ---------------------------------------------------- image sources */
typedef struct {
  v3 pos;
  double dist;
  double energy[RO_BANDS], mult[RO_BANDS];
  int64_t ray_count;
  int32_t order;
  const int32_t* path; /* points into the caller's history (len = order) */
  int has_proj;
  v3 proj;
} img_t;

struct ro_images {
  img_t* im;
  int64_t n;
  int32_t* paths; /* owned copies */
};

typedef struct {
  const int64_t* off;
  const int32_t* h;
} path_ctx;

static _Thread_local path_ctx g_pc;
static _Thread_local const double* g_pts;

/* std::lexicographical_compare on face paths */
static int path_cmp(const int32_t* a, int64_t la, const int32_t* b, int64_t lb) {
  int64_t m = la < lb ? la : lb;
  for (int64_t i = 0; i < m; ++i)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  if (la != lb) return la < lb ? -1 : 1;
  return 0;
}

static int group_cmp(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  int c = path_cmp(g_pc.h + g_pc.off[a], g_pc.off[a + 1] - g_pc.off[a],
                   g_pc.h + g_pc.off[b], g_pc.off[b + 1] - g_pc.off[b]);
  if (c) return c;
  return a < b ? -1 : (a > b); /* std::map keeps insertion order in a group */
}

static int lexpt_cmp(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  const double* x = g_pts + 3 * a;
  const double* y = g_pts + 3 * b;
  for (int k = 0; k < 3; ++k)
    if (x[k] != y[k]) return x[k] < y[k] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

typedef struct {
  img_t* v;
  int64_t n, cap;
} imgvec;

static void iv_push(imgvec* v, const img_t* x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 256;
    v->v = (img_t*)realloc(v->v, sizeof(img_t) * v->cap);
  }
  v->v[v->n++] = *x;
}

/* make_image image_sources.cpp:15-25 over members idx[0..m) */
static img_t make_image(const int64_t* idx, int64_t m, const double* retro,
                        const double* mult, const int64_t* off, const int32_t* h) {
  img_t im;
  memset(&im, 0, sizeof im);
  v3 sum = mk(0.0, 0.0, 0.0);
  for (int64_t i = 0; i < m; ++i)
    sum = vadd(sum, mk(retro[3 * idx[i]], retro[3 * idx[i] + 1], retro[3 * idx[i] + 2]));
  im.pos = vdiv(sum, (double)m);
  im.ray_count = m;
  im.path = h + off[idx[0]];
  im.order = (int32_t)(off[idx[0] + 1] - off[idx[0]]);
  memcpy(im.mult, mult + RO_BANDS * idx[0], sizeof(double) * RO_BANDS);
  return im;
}

/* split_group image_sources.cpp:28-65 */
static void split_group(int64_t* idx, int64_t m, double tol, const double* retro,
                        const double* mult, const int64_t* off, const int32_t* h,
                        imgvec* out) {
  v3 mean = mk(0.0, 0.0, 0.0);
  for (int64_t i = 0; i < m; ++i)
    mean = vadd(mean, mk(retro[3 * idx[i]], retro[3 * idx[i] + 1], retro[3 * idx[i] + 2]));
  mean = vdiv(mean, (double)m);
  double spread = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    v3 p = mk(retro[3 * idx[i]], retro[3 * idx[i] + 1], retro[3 * idx[i] + 2]);
    spread = smax(spread, vnorm(vsub(p, mean)));
  }
  if (spread <= tol) {
    img_t im = make_image(idx, m, retro, mult, off, h);
    iv_push(out, &im);
    return;
  }
  g_pts = retro;
  qsort(idx, m, sizeof(int64_t), lexpt_cmp);
  int64_t b0 = 0;
  v3 anchor = mk(retro[3 * idx[0]], retro[3 * idx[0] + 1], retro[3 * idx[0] + 2]);
  for (int64_t i = 0; i < m; ++i) {
    v3 p = mk(retro[3 * idx[i]], retro[3 * idx[i] + 1], retro[3 * idx[i] + 2]);
    if (i > b0 && vnorm(vsub(p, anchor)) > tol) {
      img_t im = make_image(idx + b0, i - b0, retro, mult, off, h);
      iv_push(out, &im);
      b0 = i;
    }
    if (i == b0) anchor = p;
  }
  img_t im = make_image(idx + b0, m - b0, retro, mult, off, h);
  iv_push(out, &im);
}

/* grid neighbour lists for the coplanar merge (exact restatement of the
 * O(I^2) greedy at image_sources.cpp:99-128: a claim needs distance <= tol,
 * so only points in adjacent cells of a (2*tol)-grid can qualify) */
typedef struct {
  int64_t cx, cy, cz;
  int64_t i;
} cell_t;

static int cell_cmp(const void* pa, const void* pb) {
  const cell_t* a = (const cell_t*)pa;
  const cell_t* b = (const cell_t*)pb;
  if (a->cx != b->cx) return a->cx < b->cx ? -1 : 1;
  if (a->cy != b->cy) return a->cy < b->cy ? -1 : 1;
  if (a->cz != b->cz) return a->cz < b->cz ? -1 : 1;
  return a->i < b->i ? -1 : (a->i > b->i);
}

static int64_t lower_cell(const cell_t* c, int64_t n, int64_t x, int64_t y, int64_t z) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    const cell_t* m = c + mid;
    int less = m->cx != x ? m->cx < x : (m->cy != y ? m->cy < y : m->cz < z);
    if (less)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

static int i64_cmp(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y);
}

static void merge_coplanar(imgvec* v, double tol) {
  int64_t n = v->n;
  if (n == 0) return;
  double cs = 2.0 * tol;
  cell_t* cells = (cell_t*)malloc(sizeof(cell_t) * n);
  for (int64_t i = 0; i < n; ++i) {
    cells[i].cx = (int64_t)floor(v->v[i].pos.x / cs);
    cells[i].cy = (int64_t)floor(v->v[i].pos.y / cs);
    cells[i].cz = (int64_t)floor(v->v[i].pos.z / cs);
    cells[i].i = i;
  }
  qsort(cells, n, sizeof(cell_t), cell_cmp);
  char* used = (char*)calloc(n, 1);
  int64_t* cand = NULL;
  int64_t ncap = 0;
  imgvec out = {0};
  for (int64_t i = 0; i < n; ++i) {
    if (used[i]) continue;
    img_t acc = v->v[i];
    const img_t* vi = v->v + i;
    v3 weighted = vscale((double)acc.ray_count, acc.pos); /* position * ray_count */
    weighted = mk(acc.pos.x * (double)acc.ray_count, acc.pos.y * (double)acc.ray_count,
                  acc.pos.z * (double)acc.ray_count);
    int64_t cx = (int64_t)floor(vi->pos.x / cs), cy = (int64_t)floor(vi->pos.y / cs),
            cz = (int64_t)floor(vi->pos.z / cs);
    int64_t nc = 0;
    for (int64_t dx = -1; dx <= 1; ++dx)
      for (int64_t dy = -1; dy <= 1; ++dy)
        for (int64_t dz = -1; dz <= 1; ++dz) {
          int64_t p = lower_cell(cells, n, cx + dx, cy + dy, cz + dz);
          for (; p < n && cells[p].cx == cx + dx && cells[p].cy == cy + dy &&
                 cells[p].cz == cz + dz;
               ++p) {
            if (cells[p].i <= i) continue;
            if (nc == ncap) {
              ncap = ncap ? 2 * ncap : 64;
              cand = (int64_t*)realloc(cand, sizeof(int64_t) * ncap);
            }
            cand[nc++] = cells[p].i;
          }
        }
    qsort(cand, nc, sizeof(int64_t), i64_cmp);
    for (int64_t c = 0; c < nc; ++c) {
      int64_t j = cand[c];
      if (used[j]) continue;
      const img_t* o = v->v + j;
      if (o->order != acc.order) continue;
      if (vnorm(vsub(o->pos, vi->pos)) > tol) continue;
      int bad = 0;
      for (int b = 0; b < RO_BANDS; ++b)
        if (fabs(o->mult[b] - acc.mult[b]) > 1e-12) bad = 1;
      if (bad) continue;
      weighted = vadd(weighted, mk(o->pos.x * (double)o->ray_count, o->pos.y * (double)o->ray_count,
                                   o->pos.z * (double)o->ray_count));
      acc.ray_count += o->ray_count;
      if (path_cmp(o->path, o->order, acc.path, acc.order) < 0) acc.path = o->path;
      used[j] = 1;
    }
    acc.pos = vdiv(weighted, (double)acc.ray_count);
    iv_push(&out, &acc);
  }
  free(cand);
  free(used);
  free(cells);
  free(v->v);
  *v = out;
}

static int final_cmp(const void* pa, const void* pb) {
  const img_t* a = (const img_t*)pa;
  const img_t* b = (const img_t*)pb;
  if (a->order != b->order) return a->order < b->order ? -1 : 1;
  if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
  return path_cmp(a->path, a->order, b->path, b->order);
}

ro_images* ro_image_sources(const ro_scene* s, int64_t n, const int32_t* ray,
                            const double* point, const double* dir,
                            const double* path, const double* mult,
                            const int64_t* hist_off, const int32_t* hist,
                            int64_t total_rays, const double* air4,
                            const double* recv, double tol_scale,
                            int merge_coplanar_flag) {
  (void)ray;
  double beta[RO_BANDS];
  if (ro_air_beta_bands(air4, beta)) return NULL;
  double blo[3], bhi[3];
  ro_scene_bounds(s, blo, bhi);
  double diag = vnorm(mk(bhi[0] - blo[0], bhi[1] - blo[1], bhi[2] - blo[2]));
  double tol = tol_scale * diag;
  /* retro_propagate image_sources.cpp:9-11 */
  double* retro = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k)
      retro[3 * i + k] = point[3 * i + k] - path[i] * dir[3 * i + k];
  /* cluster image_sources.cpp:82-132: std::map over exact face paths */
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  g_pc.off = hist_off;
  g_pc.h = hist;
  qsort(idx, n, sizeof(int64_t), group_cmp);
  imgvec v = {0};
  for (int64_t g0 = 0; g0 < n;) {
    int64_t g1 = g0 + 1;
    while (g1 < n && path_cmp(hist + hist_off[idx[g0]], hist_off[idx[g0] + 1] - hist_off[idx[g0]],
                              hist + hist_off[idx[g1]], hist_off[idx[g1] + 1] - hist_off[idx[g1]]) == 0)
      ++g1;
    split_group(idx + g0, g1 - g0, tol, retro, mult, hist_off, hist, &v);
    g0 = g1;
  }
  if (merge_coplanar_flag) merge_coplanar(&v, tol);
  /* attach_energy :134-140, project :142-152 */
  v3 rc = mk(recv[0], recv[1], recv[2]);
  for (int64_t i = 0; i < v.n; ++i) {
    img_t* im = v.v + i;
    im->dist = vnorm(vsub(im->pos, rc));
    double frac = (double)im->ray_count / (double)total_rays;
    for (int b = 0; b < RO_BANDS; ++b)
      im->energy[b] = (frac * exp((-beta[b]) * im->dist)) * im->mult[b];
    im->has_proj = 0;
    if (im->order >= 1) {
      v3 tw = vsub(im->pos, rc);
      double dd = vnorm(tw);
      if (dd != 0.0) {
        hit_t h = nearest_hit(s, rc, vdiv(tw, dd), NULL, NULL);
        if (h.ok) {
          im->has_proj = 1;
          im->proj = h.point;
        }
      }
    }
  }
  qsort(v.v, v.n, sizeof(img_t), final_cmp);
  ro_images* r = (ro_images*)calloc(1, sizeof(ro_images));
  r->n = v.n;
  r->im = v.v;
  int64_t tp = 0;
  for (int64_t i = 0; i < v.n; ++i) tp += v.v[i].order;
  r->paths = (int32_t*)malloc(sizeof(int32_t) * (tp > 0 ? tp : 1));
  int64_t off = 0;
  for (int64_t i = 0; i < v.n; ++i) {
    memcpy(r->paths + off, v.v[i].path, sizeof(int32_t) * v.v[i].order);
    v.v[i].path = r->paths + off;
    off += v.v[i].order;
  }
  free(retro);
  free(idx);
  return r;
}

void ro_images_info(const ro_images* r, int64_t* n, int64_t* total_path) {
  *n = r->n;
  int64_t tp = 0;
  for (int64_t i = 0; i < r->n; ++i) tp += r->im[i].order;
  *total_path = tp;
}

void ro_images_get(const ro_images* r, double* pos, double* dist,
                   double* energy, double* mult, int32_t* ray_count,
                   int32_t* order, int32_t* has_proj, double* proj,
                   int64_t* path_off, int32_t* path) {
  int64_t off = 0;
  for (int64_t i = 0; i < r->n; ++i) {
    const img_t* im = r->im + i;
    pos[3 * i] = im->pos.x;
    pos[3 * i + 1] = im->pos.y;
    pos[3 * i + 2] = im->pos.z;
    dist[i] = im->dist;
    memcpy(energy + RO_BANDS * i, im->energy, sizeof(double) * RO_BANDS);
    memcpy(mult + RO_BANDS * i, im->mult, sizeof(double) * RO_BANDS);
    ray_count[i] = (int32_t)im->ray_count;
    order[i] = im->order;
    has_proj[i] = im->has_proj;
    proj[3 * i] = im->has_proj ? im->proj.x : 0.0;
    proj[3 * i + 1] = im->has_proj ? im->proj.y : 0.0;
    proj[3 * i + 2] = im->has_proj ? im->proj.z : 0.0;
    path_off[i] = off;
    memcpy(path + off, im->path, sizeof(int32_t) * im->order);
    off += im->order;
  }
  path_off[r->n] = off;
}

void ro_images_free(ro_images* r) {
  if (!r) return;
  free(r->im);
  free(r->paths);
  free(r);
}

/* ---------------------------------------------------- air absorption
 * AirModel::validate air_absorption.cpp:8-19, air_alpha_db_per_m :21-53 */
static const double kCenters[RO_BANDS] = {62.5, 125.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0, 8000.0};

static int air_validate(const double* a) {
  if (a[0] == 0.0) return 0;
  if (a[1] < -20.0 || a[1] > 50.0) {
    set_err("air temperature outside [-20, 50] C");
    return 1;
  }
  if (a[2] < 10.0 || a[2] > 100.0) {
    set_err("relative humidity outside [10, 100] %");
    return 1;
  }
  if (a[3] < 80.0 || a[3] > 120.0) {
    set_err("pressure outside [80, 120] kPa");
    return 1;
  }
  return 0;
}

double ro_air_alpha(const double* a, double f) {
  if (a[0] == 0.0) return 0.0;
  const double tk = a[1] + 273.15;
  const double t_rel = tk / 293.15;
  const double p_rel = a[3] / 101.325;
  const double c_sat = -6.8346 * pow(273.16 / tk, 1.261) + 4.6151;
  const double h = a[2] * pow(10.0, c_sat) / p_rel;
  const double fro = p_rel * (24.0 + 4.04e4 * h * (0.02 + h) / (0.391 + h));
  const double frn = p_rel * pow(t_rel, -0.5) *
                     (9.0 + 280.0 * h * exp(-4.170 * (pow(t_rel, -1.0 / 3.0) - 1.0)));
  const double f2 = f * f;
  const double classical = 1.84e-11 / p_rel * sqrt(t_rel);
  const double relax = pow(t_rel, -2.5) *
                       (0.01275 * exp(-2239.1 / tk) / (fro + f2 / fro) +
                        0.1068 * exp(-3352.0 / tk) / (frn + f2 / frn));
  return 8.686 * f2 * (classical + relax);
}

/* air_beta / air_beta_bands :55-65 */
int ro_air_beta_bands(const double* a, double* beta) {
  if (air_validate(a)) return 1;
  for (int b = 0; b < RO_BANDS; ++b) beta[b] = ro_air_alpha(a, kCenters[b]) * log(10.0) / 10.0;
  return 0;
}

/* ---------------------------------------------------- IR synthesis */
/* design_band_filter rir.cpp:32-58, taps parameterised (reference: 1023) */
int ro_band_filter(int band, double fs, int taps, double* out) {
  if (band < 0 || band >= RO_BANDS) {
    set_err("band index out of range");
    return 1;
  }
  const double fl = kCenters[band] / sqrt(2.0);
  const double fh = kCenters[band] * sqrt(2.0);
  if (fs < 2.0 * fh) {
    set_err("sample rate too low for the top band edge");
    return 1;
  }
  const int delay = (taps - 1) / 2;
  for (int n = 0; n < taps; ++n) {
    const int m = n - delay;
    double ideal;
    if (m == 0)
      ideal = 2.0 * (fh - fl) / fs;
    else
      ideal = (sin(2.0 * M_PI * fh * m / fs) - sin(2.0 * M_PI * fl * m / fs)) / (M_PI * m);
    const double hann = 0.5 * (1.0 - cos(2.0 * M_PI * n / (taps - 1)));
    out[n] = ideal * hann;
  }
  return 0;
}

typedef struct {
  double t, a;
} ev_t;

static int ev_cmp(const void* pa, const void* pb) {
  const ev_t* x = (const ev_t*)pa;
  const ev_t* y = (const ev_t*)pb;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  if (x->a != y->a) return x->a < y->a ? -1 : 1;
  return 0;
}

/* build_pulse_trains rir.cpp:9-30 + synthesize rir.cpp:60-96 */
int64_t ro_synthesize(int64_t n, const double* dist, const double* energy,
                      double c, double fs, int taps, int32_t band_mask,
                      double* out, int64_t cap) {
  if (c <= 0.0) {
    set_err("speed of sound must be > 0");
    return -1;
  }
  ev_t* ev = (ev_t*)malloc(sizeof(ev_t) * (n > 0 ? n : 1));
  double last = 0.0;
  int any = 0;
  for (int64_t i = 0; i < n; ++i) {
    double t = dist[i] / c;
    if (t < 0.0) {
      free(ev);
      set_err("pulse events cannot precede t = 0");
      return -1;
    }
  }
  /* all bands carry one event per image at the same time */
  for (int b = 0; b < RO_BANDS; ++b)
    if (band_mask & (1 << b))
      for (int64_t i = 0; i < n; ++i) {
        last = smax(last, dist[i] / c);
        any = 1;
      }
  if (!any) {
    free(ev);
    return 0;
  }
  const int delay = (taps - 1) / 2;
  const int64_t length = (int64_t)llround(last * fs) + delay + 1;
  double* samples = (double*)calloc(length, sizeof(double));
  double* kern = (double*)malloc(sizeof(double) * taps);
  for (int b = 0; b < RO_BANDS; ++b) {
    if (!(band_mask & (1 << b))) continue;
    if (ro_band_filter(b, fs, taps, kern)) {
      free(ev);
      free(samples);
      free(kern);
      return -1;
    }
    for (int64_t i = 0; i < n; ++i) {
      ev[i].t = dist[i] / c;
      ev[i].a = sqrt(energy[RO_BANDS * i + b]);
    }
    qsort(ev, n, sizeof(ev_t), ev_cmp);
    for (int64_t i = 0; i < n; ++i) {
      const long center = lround(ev[i].t * fs);
      for (int k = 0; k < taps; ++k) {
        const long j = center + k - delay;
        if (j < 0) continue;
        if (j >= (long)length) break;
        samples[j] += ev[i].a * kern[k];
      }
    }
  }
  if (out) memcpy(out, samples, sizeof(double) * (length < cap ? length : cap));
  free(ev);
  free(samples);
  free(kern);
  return length;
}

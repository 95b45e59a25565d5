/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see sg_oracle.h for the contract).
 *
 * Plain-C restatement of the reference hot path. Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Compiled with -ffp-contract=off so each source operation rounds once, like
 * the reference's scalar code.
 *
 * Third-party arithmetic restated here: Eigen >= 3.3 (version unpinned by the
 * reference, proj/CMakeLists.txt:13) — Quaternion product, AngleAxis->
 * Quaternion and Quaternion*Vector3 (`uv = u x v; uv += uv; v + w*uv + u x uv`)
 * follow Eigen's published Geometry/Quaternion.h formulas; glibc libm for
 * log/cos/sin/sqrt.
 *
 * Compiler semantics pinned: the reference builds with g++ (CMake default on
 * this Linux image). g++ evaluates constructor arguments right-to-left (see
 * oracle/probe_eval_order.cpp), so in `Eigen::Vector3d(rng.normal(..),
 * rng.normal(..), rng.normal(..))` (envs.cpp:232-234) the FIRST draw lands in
 * z and the LAST in x. This file reproduces that order explicitly.
 */
#define _GNU_SOURCE
#include "sg_oracle.h"

#include <ctype.h>
#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#ifndef SGO_REAL
#define SGO_REAL double
#endif
typedef SGO_REAL real;

#define SGO_SIN(x) (sizeof(real) == sizeof(float) ? (real)sinf((float)(x)) : (real)sin((double)(x)))
#define SGO_COS(x) (sizeof(real) == sizeof(float) ? (real)cosf((float)(x)) : (real)cos((double)(x)))
#define SGO_SQRT(x) (sizeof(real) == sizeof(float) ? (real)sqrtf((float)(x)) : (real)sqrt((double)(x)))
#define SGO_ACOS(x) (sizeof(real) == sizeof(float) ? (real)acosf((float)(x)) : (real)acos((double)(x)))

/* ======================================================================
 * PCG32 — rng.hpp:25-83
 * ====================================================================== */
uint32_t sgo_pcg32_next(sgo_pcg32* r) { /* rng.hpp:38-44 */
  uint64_t old = r->state;
  r->state = old * 6364136223846793005ULL + r->inc;
  uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = (uint32_t)(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

void sgo_pcg32_seed(sgo_pcg32* r, uint64_t initstate, uint64_t initseq) { /* rng.hpp:30-36 */
  r->state = 0u;
  r->inc = (initseq << 1u) | 1u;
  sgo_pcg32_next(r);
  r->state += initstate;
  sgo_pcg32_next(r);
}

static double next_double(sgo_pcg32* r) { return sgo_pcg32_next(r) * 0x1.0p-32; } /* rng.hpp:47 */

double sgo_pcg32_uniform(sgo_pcg32* r, double lo, double hi) { /* rng.hpp:49 */
  return lo + (hi - lo) * next_double(r);
}

double sgo_pcg32_normal(sgo_pcg32* r) { /* rng.hpp:53-57 */
  double u1 = (sgo_pcg32_next(r) + 0.5) * 0x1.0p-32;
  double u2 = next_double(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586477 * u2);
}

static uint64_t splitmix64(uint64_t* x) { /* rng.hpp:69-75 */
  *x += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void sgo_make_stream(uint64_t seed, uint64_t stream_id, sgo_pcg32* out) { /* rng.hpp:78-83 */
  uint64_t x = seed ^ (0x2545f4914f6cdd1dULL * (stream_id + 1));
  uint64_t initstate = splitmix64(&x);
  uint64_t initseq = splitmix64(&x);
  sgo_pcg32_seed(out, initstate, initseq);
}

void sgo_fill_uniform_actions(sgo_pcg32* r, double* a, int64_t count) { /* bench.cpp:31-35 */
  for (int64_t k = 0; k < count; ++k) a[k] = sgo_pcg32_uniform(r, -1.0, 1.0);
}

/* the trainer's per-step noise: one serial stream, row-major (ppo.cpp:264-270) */
void sgo_fill_normals(sgo_pcg32* r, double* z, int64_t count) {
  for (int64_t k = 0; k < count; ++k) z[k] = sgo_pcg32_normal(r);
}

/* ======================================================================
 * Quaternion / vector helpers with Eigen semantics (geometry.hpp:25-49)
 * ====================================================================== */
#define DEFINE_GEOM(T, SUF, SINF, COSF)                                                          \
  static void qmul_##SUF(const T* a, const T* b, T* o) {                                       \
    T w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];                               \
    T x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];                               \
    T y = a[0] * b[2] + a[2] * b[0] + a[3] * b[1] - a[1] * b[3];                               \
    T z = a[0] * b[3] + a[3] * b[0] + a[1] * b[2] - a[2] * b[1];                               \
    o[0] = w; o[1] = x; o[2] = y; o[3] = z;                                                    \
  }                                                                                            \
  static void cross_##SUF(const T* a, const T* b, T* o) {                                      \
    T x = a[1] * b[2] - a[2] * b[1];                                                           \
    T y = a[2] * b[0] - a[0] * b[2];                                                           \
    T z = a[0] * b[1] - a[1] * b[0];                                                           \
    o[0] = x; o[1] = y; o[2] = z;                                                              \
  }                                                                                            \
  /* Eigen _transformVector: uv = u x v; uv += uv; v + w*uv + u x uv */                        \
  static void qrot_##SUF(const T* q, const T* v, T* o) {                                       \
    T u[3] = {q[1], q[2], q[3]}, uv[3], c[3];                                                  \
    cross_##SUF(u, v, uv);                                                                     \
    uv[0] += uv[0]; uv[1] += uv[1]; uv[2] += uv[2];                                            \
    cross_##SUF(u, uv, c);                                                                     \
    T r0 = v[0] + q[0] * uv[0] + c[0];                                                         \
    T r1 = v[1] + q[0] * uv[1] + c[1];                                                         \
    T r2 = v[2] + q[0] * uv[2] + c[2];                                                         \
    o[0] = r0; o[1] = r1; o[2] = r2;                                                           \
  }                                                                                            \
  /* AngleAxis -> Quaternion: w = cos(a/2), v = sin(a/2) * axis */                             \
  static void qaa_##SUF(T angle, const T* axis, T* o) {                                        \
    T ha = (T)0.5 * angle;                                                                     \
    T s = SINF(ha);                                                                            \
    o[0] = COSF(ha); o[1] = s * axis[0]; o[2] = s * axis[1]; o[3] = s * axis[2];               \
  }

DEFINE_GEOM(double, d, sin, cos)
DEFINE_GEOM(real, r, SGO_SIN, SGO_COS)

/* quat_from_rpy: AA(yaw,Z) * AA(pitch,Y) * AA(roll,X)  (geometry.hpp:45-49) */
static void quat_from_rpy(double roll, double pitch, double yaw, double* o) {
  const double ez[3] = {0, 0, 1}, ey[3] = {0, 1, 0}, ex[3] = {1, 0, 0};
  double qz[4], qy[4], qx[4], t[4];
  qaa_d(yaw, ez, qz);
  qaa_d(pitch, ey, qy);
  qaa_d(roll, ex, qx);
  qmul_d(qz, qy, t);
  qmul_d(t, qx, o);
}

/* ======================================================================
 * Descriptor parser — robot_model.cpp:39-283
 * ====================================================================== */
static void seterr(char* err, int errlen, const char* fmt, ...) {
  if (!err || errlen <= 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, (size_t)errlen, fmt, ap);
  va_end(ap);
}

static char* trim(char* s) { /* robot_model.cpp:39-44 */
  while (*s == ' ' || *s == '\t' || *s == '\r') ++s;
  size_t n = strlen(s);
  while (n > 0 && (s[n - 1] == ' ' || s[n - 1] == '\t' || s[n - 1] == '\r')) s[--n] = 0;
  return s;
}

/* robot_model.cpp:46-59: exactly `expect` numbers and nothing else, with the
 * number grammar of formatted stream extraction (`in >> double`, libstdc++
 * num_get in the "C" locale): [sign] digits [. digits] [(e|E) [sign] digits],
 * greedy; no inf / nan / hex. A token that runs to the end of the value ends
 * the read with eof set (a malformed tail such as a lone "-" or "1e" is then
 * dropped, not an error); a malformed token before the end is an error. */
static int parse_numbers(const char* v, int expect, double* out) {
  const char* p = v;
  int n = 0;
  for (;;) {
    while (isspace((unsigned char)*p)) ++p;
    if (!*p) return n == expect;
    const char* s = p;
    int mant = 0, has_e = 0, expd = 0;
    if (*p == '+' || *p == '-') ++p;
    while (isdigit((unsigned char)*p)) ++p, ++mant;
    if (*p == '.') {
      ++p;
      while (isdigit((unsigned char)*p)) ++p, ++mant;
    }
    if (mant && (*p == 'e' || *p == 'E')) {
      has_e = 1;
      ++p;
      if (*p == '+' || *p == '-') ++p;
      while (isdigit((unsigned char)*p)) ++p, ++expd;
    }
    const int valid = mant > 0 && (!has_e || expd > 0);
    const int at_end = *p == 0;
    if (!valid) return at_end ? n == expect : 0;
    char buf[128];
    size_t len = (size_t)(p - s);
    if (len >= sizeof(buf)) return 0;
    memcpy(buf, s, len);
    buf[len] = 0;
    if (n < expect) out[n] = strtod(buf, NULL);
    ++n;
    if (at_end) return n == expect;
  }
}

#define MAX_FIELDS 24
typedef struct {
  int line;
  int active;
  int n;
  char key[MAX_FIELDS][64];
  char val[MAX_FIELDS][256];
  int lines[MAX_FIELDS];
} pending_joint;

static int take(pending_joint* pj, const char* key, char** val, int* line) {
  for (int i = 0; i < pj->n; ++i) {
    if (pj->key[i][0] && strcmp(pj->key[i], key) == 0) {
      *val = pj->val[i];
      *line = pj->lines[i];
      pj->key[i][0] = 0;
      return 1;
    }
  }
  return 0;
}

/* robot_model.cpp:81-131 */
static int flush_joint(pending_joint* pj, int index, const char* origin, sgo_joint* j, char* err,
                       int errlen) {
  char* v;
  int l;
  memset(j, 0, sizeof(*j));
  j->axis[2] = 1.0;
  j->origin_quat[0] = 1.0;
#define REQUIRE_FIELD(k)                                                                          \
  if (!take(pj, k, &v, &l)) {                                                                     \
    seterr(err, errlen, "%s:%d: joint #%d is missing required field '%s'", origin, pj->line, index, \
           k);                                                                                    \
    return 2;                                                                                     \
  }
#define NUMS(k, cnt, dst)                                                                  \
  if (!parse_numbers(v, cnt, dst)) {                                                       \
    seterr(err, errlen, "%s:%d: field '%s' expects %d number(s), got '%s'", origin, l, k, cnt, v); \
    return 2;                                                                              \
  }
  REQUIRE_FIELD("name");
  snprintf(j->name, sizeof(j->name), "%s", v);
  REQUIRE_FIELD("kind");
  if (strcmp(v, "revolute") == 0) j->kind = SGO_REVOLUTE;
  else if (strcmp(v, "prismatic") == 0) j->kind = SGO_PRISMATIC;
  else if (strcmp(v, "fixed") == 0) j->kind = SGO_FIXED;
  else {
    seterr(err, errlen, "%s:%d: unknown joint kind '%s'", origin, l, v);
    return 2;
  }
  if (take(pj, "axis", &v, &l)) {
    NUMS("axis", 3, j->axis);
  } else if (j->kind != SGO_FIXED) {
    seterr(err, errlen, "%s:%d: joint #%d is missing required field 'axis'", origin, pj->line, index);
    return 2;
  }
  REQUIRE_FIELD("origin_xyz");
  NUMS("origin_xyz", 3, j->origin_xyz);
  REQUIRE_FIELD("origin_rpy");
  double rpy[3];
  NUMS("origin_rpy", 3, rpy);
  quat_from_rpy(rpy[0], rpy[1], rpy[2], j->origin_quat);
  if (j->kind != SGO_FIXED) {
    double lim[2];
    REQUIRE_FIELD("limits");
    NUMS("limits", 2, lim);
    j->limit_lo = lim[0];
    j->limit_hi = lim[1];
    REQUIRE_FIELD("velocity_limit");
    NUMS("velocity_limit", 1, &j->velocity_limit);
    REQUIRE_FIELD("effort_limit");
    NUMS("effort_limit", 1, &j->effort_limit);
  }
  /* unknown field: std::map iteration -> lexicographically first leftover key */
  int first = -1;
  for (int i = 0; i < pj->n; ++i)
    if (pj->key[i][0] && (first < 0 || strcmp(pj->key[i], pj->key[first]) < 0)) first = i;
  if (first >= 0) {
    seterr(err, errlen, "%s:%d: unknown joint field '%s'", origin, pj->lines[first], pj->key[first]);
    return 2;
  }
  memset(pj, 0, sizeof(*pj));
  return 0;
#undef REQUIRE_FIELD
#undef NUMS
}

static int validate_model(const sgo_robot* m, const char* origin, char* err, int errlen) {
  /* robot_model.cpp:133-161 */
  if (!m->name[0]) { seterr(err, errlen, "%s: missing robot name", origin); return 2; }
  if (m->n_joints == 0) { seterr(err, errlen, "%s: robot has no joints", origin); return 2; }
  for (int i = 0; i < m->n_joints; ++i) {
    const sgo_joint* j = &m->joints[i];
    if (j->kind == SGO_FIXED) continue;
    double nrm = sqrt(j->axis[0] * j->axis[0] + j->axis[1] * j->axis[1] + j->axis[2] * j->axis[2]);
    if (fabs(nrm - 1.0) > 1e-12) {
      seterr(err, errlen, "%s: joint '%s': axis is not unit-norm", origin, j->name);
      return 2;
    }
    if (!(j->limit_lo < j->limit_hi)) {
      seterr(err, errlen, "%s: joint '%s': limit_lo must be < limit_hi", origin, j->name);
      return 2;
    }
    if (!(j->velocity_limit > 0.0)) {
      seterr(err, errlen, "%s: joint '%s': velocity_limit must be > 0", origin, j->name);
      return 2;
    }
    if (!(j->effort_limit > 0.0)) {
      seterr(err, errlen, "%s: joint '%s': effort_limit must be > 0", origin, j->name);
      return 2;
    }
  }
  if (m->jaw_joint >= 0 || m->jaw_joint < -1) {
    int idx = m->jaw_joint;
    if (idx < 0 || idx >= m->n_joints) {
      seterr(err, errlen, "%s: jaw joint index out of range", origin);
      return 2;
    }
    if (m->joints[idx].kind != SGO_REVOLUTE) {
      seterr(err, errlen, "%s: jaw joint '%s' must be revolute", origin, m->joints[idx].name);
      return 2;
    }
  }
  return 0;
}

int sgo_parse_robot(const char* text, const char* origin, sgo_robot* m, char* err, int errlen) {
  /* robot_model.cpp:191-283 */
  memset(m, 0, sizeof(*m));
  m->tip_quat[0] = 1.0;
  m->jaw_joint = -1;
  pending_joint* pj = (pending_joint*)calloc(1, sizeof(pending_joint));
  char section[64] = "";
  int have_tool_tip = 0, line_no = 0, rc = 0;
  const char* p = text;
  char raw[1024];
  while (*p) {
    const char* nl = strchr(p, '\n');
    size_t len = nl ? (size_t)(nl - p) : strlen(p);
    if (len >= sizeof(raw)) len = sizeof(raw) - 1;
    memcpy(raw, p, len);
    raw[len] = 0;
    p = nl ? nl + 1 : p + strlen(p);
    ++line_no;
    char* line = trim(raw);
    if (!line[0] || line[0] == '#') continue;
    size_t ll = strlen(line);
    if (line[0] == '[') {
      if (line[ll - 1] != ']') { seterr(err, errlen, "%s:%d: malformed section header", origin, line_no); rc = 2; goto done; }
      if (strcmp(section, "joint") == 0 && pj->active) {
        if (m->n_joints >= SGO_MAX_JOINTS) { seterr(err, errlen, "%s: too many joints", origin); rc = 2; goto done; }
        rc = flush_joint(pj, m->n_joints, origin, &m->joints[m->n_joints], err, errlen);
        if (rc) goto done;
        m->n_joints++;
      }
      line[ll - 1] = 0;
      snprintf(section, sizeof(section), "%s", line + 1);
      if (strcmp(section, "robot") && strcmp(section, "joint") && strcmp(section, "tool_tip") &&
          strcmp(section, "jaw")) {
        seterr(err, errlen, "%s:%d: unknown section [%s]", origin, line_no, section);
        rc = 2;
        goto done;
      }
      if (strcmp(section, "joint") == 0) {
        memset(pj, 0, sizeof(*pj));
        pj->active = 1;
        pj->line = line_no;
      }
      continue;
    }
    char* eq = strchr(line, '=');
    if (!eq) { seterr(err, errlen, "%s:%d: expected 'key = value'", origin, line_no); rc = 2; goto done; }
    *eq = 0;
    char* key = trim(line);
    char* value = trim(eq + 1);
    if (!key[0] || !value[0]) { seterr(err, errlen, "%s:%d: expected 'key = value'", origin, line_no); rc = 2; goto done; }
    double nums[3];
    if (strcmp(section, "robot") == 0) {
      if (strcmp(key, "name") == 0) {
        snprintf(m->name, sizeof(m->name), "%s", value);
      } else if (strcmp(key, "format_version") == 0) {
        if (!parse_numbers(value, 1, nums)) { seterr(err, errlen, "%s:%d: field '%s' expects 1 number(s), got '%s'", origin, line_no, key, value); rc = 2; goto done; }
        if ((int)nums[0] != 1) { seterr(err, errlen, "%s:%d: unsupported format_version %d", origin, line_no, (int)nums[0]); rc = 2; goto done; }
      } else {
        seterr(err, errlen, "%s:%d: unknown [robot] field '%s'", origin, line_no, key);
        rc = 2;
        goto done;
      }
    } else if (strcmp(section, "joint") == 0) {
      for (int i = 0; i < pj->n; ++i)
        if (strcmp(pj->key[i], key) == 0) { seterr(err, errlen, "%s:%d: duplicate field '%s'", origin, line_no, key); rc = 2; goto done; }
      if (pj->n >= MAX_FIELDS) { seterr(err, errlen, "%s:%d: too many fields", origin, line_no); rc = 2; goto done; }
      snprintf(pj->key[pj->n], 64, "%s", key);
      snprintf(pj->val[pj->n], 256, "%s", value);
      pj->lines[pj->n] = line_no;
      pj->n++;
    } else if (strcmp(section, "tool_tip") == 0) {
      have_tool_tip = 1;
      if (strcmp(key, "xyz") == 0) {
        if (!parse_numbers(value, 3, m->tip_xyz)) { seterr(err, errlen, "%s:%d: field '%s' expects 3 number(s), got '%s'", origin, line_no, key, value); rc = 2; goto done; }
      } else if (strcmp(key, "rpy") == 0) {
        if (!parse_numbers(value, 3, nums)) { seterr(err, errlen, "%s:%d: field '%s' expects 3 number(s), got '%s'", origin, line_no, key, value); rc = 2; goto done; }
        quat_from_rpy(nums[0], nums[1], nums[2], m->tip_quat);
      } else {
        seterr(err, errlen, "%s:%d: unknown [tool_tip] field '%s'", origin, line_no, key);
        rc = 2;
        goto done;
      }
    } else if (strcmp(section, "jaw") == 0) {
      if (strcmp(key, "joint") == 0) {
        if (!parse_numbers(value, 1, nums)) { seterr(err, errlen, "%s:%d: field '%s' expects 1 number(s), got '%s'", origin, line_no, key, value); rc = 2; goto done; }
        m->jaw_joint = (int)nums[0];
        if (m->jaw_joint == -1) m->jaw_joint = -2; /* explicit -1 is out of range */
      } else {
        seterr(err, errlen, "%s:%d: unknown [jaw] field '%s'", origin, line_no, key);
        rc = 2;
        goto done;
      }
    } else {
      seterr(err, errlen, "%s:%d: content before any section header", origin, line_no);
      rc = 2;
      goto done;
    }
  }
  if (strcmp(section, "joint") == 0 && pj->active) {
    if (m->n_joints >= SGO_MAX_JOINTS) { seterr(err, errlen, "%s: too many joints", origin); rc = 2; goto done; }
    rc = flush_joint(pj, m->n_joints, origin, &m->joints[m->n_joints], err, errlen);
    if (rc) goto done;
    m->n_joints++;
  }
  if (!have_tool_tip) { seterr(err, errlen, "%s: missing [tool_tip] section", origin); rc = 2; goto done; }
  m->dof = 0;
  for (int i = 0; i < m->n_joints; ++i)
    if (m->joints[i].kind != SGO_FIXED) m->dof_to_joint[m->dof++] = i;
  rc = validate_model(m, origin, err, errlen);
done:
  free(pj);
  return rc;
}

int sgo_jaw_dof(const sgo_robot* m) { /* robot_model.cpp:174-180 */
  if (m->jaw_joint < 0) return -1;
  for (int d = 0; d < m->dof; ++d)
    if (m->dof_to_joint[d] == m->jaw_joint) return d;
  return -1;
}

static void mid_configuration(const sgo_robot* m, double* q) { /* robot_model.cpp:182-189 */
  for (int d = 0; d < m->dof; ++d) {
    const sgo_joint* j = &m->joints[m->dof_to_joint[d]];
    q[d] = 0.5 * (j->limit_lo + j->limit_hi);
  }
}

/* ======================================================================
 * FK — robot_model.cpp:371-402 (fk_walk), geometry.hpp:32-41
 * ====================================================================== */
#define DEFINE_FK(T, SUF)                                                          \
  static void fk_##SUF(const sgo_robot* m, const T* q, T* pos, T* quat) {          \
    T p[3] = {0, 0, 0}, rot[4] = {1, 0, 0, 0}, t[4], v[3];                         \
    int d = 0;                                                                     \
    for (int i = 0; i < m->n_joints; ++i) {                                        \
      const sgo_joint* j = &m->joints[i];                                          \
      T o[3] = {(T)j->origin_xyz[0], (T)j->origin_xyz[1], (T)j->origin_xyz[2]};    \
      T oq[4] = {(T)j->origin_quat[0], (T)j->origin_quat[1], (T)j->origin_quat[2], \
                 (T)j->origin_quat[3]};                                            \
      T ax[3] = {(T)j->axis[0], (T)j->axis[1], (T)j->axis[2]};                     \
      qrot_##SUF(rot, o, v);                                                       \
      p[0] += v[0]; p[1] += v[1]; p[2] += v[2];                                    \
      qmul_##SUF(rot, oq, t);                                                      \
      memcpy(rot, t, sizeof(t));                                                   \
      if (j->kind == SGO_FIXED) continue;                                          \
      if (j->kind == SGO_REVOLUTE) {                                               \
        T aq[4];                                                                   \
        qaa_##SUF(q[d], ax, aq);                                                   \
        qmul_##SUF(rot, aq, t);                                                    \
        memcpy(rot, t, sizeof(t));                                                 \
      } else {                                                                     \
        T av[3] = {ax[0] * q[d], ax[1] * q[d], ax[2] * q[d]};                      \
        qrot_##SUF(rot, av, v);                                                    \
        p[0] += v[0]; p[1] += v[1]; p[2] += v[2];                                  \
      }                                                                            \
      ++d;                                                                         \
    }                                                                              \
    T tp[3] = {(T)m->tip_xyz[0], (T)m->tip_xyz[1], (T)m->tip_xyz[2]};              \
    T tq[4] = {(T)m->tip_quat[0], (T)m->tip_quat[1], (T)m->tip_quat[2],            \
               (T)m->tip_quat[3]};                                                 \
    qrot_##SUF(rot, tp, v);                                                        \
    pos[0] = p[0] + v[0]; pos[1] = p[1] + v[1]; pos[2] = p[2] + v[2];              \
    if (quat) qmul_##SUF(rot, tq, quat);                                           \
  }

DEFINE_FK(double, d)
DEFINE_FK(real, r)

void sgo_fk(const sgo_robot* m, const double* q, double* pos, double* quat) {
  real qr[SGO_MAX_JOINTS], pr[3], qq[4];
  for (int d = 0; d < m->dof; ++d) qr[d] = (real)q[d];
  fk_r(m, qr, pr, qq);
  for (int k = 0; k < 3; ++k) pos[k] = pr[k];
  if (quat)
    for (int k = 0; k < 4; ++k) quat[k] = qq[k];
}

/* Homogeneous-matrix oracle with Rodrigues rotations (test_robot_model.cpp:27-56). */
static void mat4_mul(const double* a, const double* b, double* o) {
  double t[16];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += a[r * 4 + k] * b[k * 4 + c];
      t[r * 4 + c] = s;
    }
  memcpy(o, t, sizeof(t));
}
static void quat_to_mat3(const double* q, double* R) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}
static void hom(const double* R, const double* t, double* M) {
  memset(M, 0, 16 * sizeof(double));
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) M[r * 4 + c] = R[r * 3 + c];
    M[r * 4 + 3] = t[r];
  }
  M[15] = 1;
}
void sgo_fk_matrix(const sgo_robot* m, const double* q, double* M) {
  double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, R[9], H[16], z3[3] = {0, 0, 0};
  hom(I, z3, M);
  int d = 0;
  for (int i = 0; i < m->n_joints; ++i) {
    const sgo_joint* j = &m->joints[i];
    quat_to_mat3(j->origin_quat, R);
    hom(R, j->origin_xyz, H);
    mat4_mul(M, H, M);
    if (j->kind == SGO_REVOLUTE) {
      const double* a = j->axis;
      double ang = q[d++], K[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0}, KK[9], Rr[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int k = 0; k < 3; ++k) s += K[r * 3 + k] * K[k * 3 + c];
          KK[r * 3 + c] = s;
        }
      for (int k = 0; k < 9; ++k) Rr[k] = I[k] + sin(ang) * K[k] + (1.0 - cos(ang)) * KK[k];
      hom(Rr, z3, H);
      mat4_mul(M, H, M);
    } else if (j->kind == SGO_PRISMATIC) {
      double t[3] = {j->axis[0] * q[d], j->axis[1] * q[d], j->axis[2] * q[d]};
      ++d;
      hom(I, t, H);
      mat4_mul(M, H, M);
    }
  }
  quat_to_mat3(m->tip_quat, R);
  hom(R, m->tip_xyz, H);
  mat4_mul(M, H, M);
}

/* ======================================================================
 * Dynamics — dynamics.cpp:69-241
 * ====================================================================== */
void sgo_default_dynamics(const sgo_robot* m, sgo_dyn* c) { /* dynamics.cpp:69-86 */
  memset(c, 0, sizeof(*c));
  c->control_dt = 0.01;
  c->substeps = 4;
  c->control_mode = SGO_POSITION;
  for (int d = 0; d < m->dof; ++d) {
    int prismatic = m->joints[m->dof_to_joint[d]].kind == SGO_PRISMATIC;
    double mass = prismatic ? 0.5 : 0.05;
    double kp = 380.0 * mass;
    c->inertia[d] = mass;
    c->kp[d] = kp;
    c->kd[d] = 2.0 * sqrt(kp * mass);
    c->damping[d] = 0.1 * c->kd[d];
  }
}

static real rescale_to_range(real a, real lo, real hi) { /* dynamics.cpp:91-95 */
  if (a >= (real)1.0) return hi;
  if (a <= (real)-1.0) return lo;
  return lo + (real)0.5 * (a + (real)1.0) * (hi - lo);
}

/* Per-row body of dynamics.cpp:127-185. Returns -1 on non-finite action, else
 * the number of saturated entries. */
static int dyn_row(const sgo_robot* m, const sgo_dyn* cfg, int jaw, real* q, real* qd, real* qt,
                   const double* a_row) {
  const real dt_sub = (real)(cfg->control_dt / cfg->substeps); /* dynamics.cpp:119 */
  int sat = 0;
  for (int d = 0; d < m->dof; ++d) {
    const sgo_joint* j = &m->joints[m->dof_to_joint[d]];
    const real lo = (real)j->limit_lo, hi = (real)j->limit_hi;
    const real vel = (real)j->velocity_limit, eff = (real)j->effort_limit;
    const real kp = (real)cfg->kp[d], kd = (real)cfg->kd[d];
    const real damping = (real)cfg->damping[d], inertia = (real)cfg->inertia[d];
    double ad = a_row[d];
    if (!isfinite(ad)) return -1;
    real a = (real)ad;
    if (a < (real)-1.0 || a > (real)1.0) {
      a = a < (real)-1.0 ? (real)-1.0 : (real)1.0;
      ++sat;
    }
    real v_target = 0, tau_cmd = 0;
    switch (cfg->control_mode) {
      case SGO_POSITION:
        qt[d] = (d == jaw) ? (a > (real)0.0 ? hi : lo) : rescale_to_range(a, lo, hi);
        break;
      case SGO_VELOCITY: v_target = rescale_to_range(a, -vel, vel); break;
      default: tau_cmd = rescale_to_range(a, -eff, eff); break;
    }
    for (int s = 0; s < cfg->substeps; ++s) {
      real tau;
      switch (cfg->control_mode) {
        case SGO_POSITION: tau = kp * (qt[d] - q[d]) - kd * qd[d]; break;
        case SGO_VELOCITY: tau = kd * (v_target - qd[d]); break;
        default: tau = tau_cmd; break;
      }
      if (tau > eff) tau = eff;
      if (tau < -eff) tau = -eff;
      qd[d] += (tau - damping * qd[d]) / inertia * dt_sub;
      if (qd[d] > vel) qd[d] = vel;
      if (qd[d] < -vel) qd[d] = -vel;
      q[d] += qd[d] * dt_sub;
      if (q[d] < lo) {
        q[d] = lo;
        qd[d] = 0;
      } else if (q[d] > hi) {
        q[d] = hi;
        qd[d] = 0;
      }
    }
  }
  return sat;
}

/* ======================================================================
 * Thread pool — thread_pool.hpp:28-143 (chunked, caller participates,
 * chunk boundaries independent of the lane count)
 * ====================================================================== */
typedef void (*chunk_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
  int lanes;
  pthread_t* workers;
  pthread_mutex_t mu;
  pthread_cond_t cv, cv_done;
  int stop;
  uint64_t gen;
  chunk_fn fn;
  void* ctx;
  int64_t n, grain, chunks;
  int64_t next, done;
} pool_t;

static void pool_run_chunks(pool_t* p) {
  for (;;) {
    int64_t c = __atomic_fetch_add(&p->next, 1, __ATOMIC_RELAXED);
    if (c >= p->chunks) break;
    int64_t b = c * p->grain, e = b + p->grain < p->n ? b + p->grain : p->n;
    p->fn(p->ctx, b, e);
    if (__atomic_add_fetch(&p->done, 1, __ATOMIC_ACQ_REL) == p->chunks) {
      pthread_mutex_lock(&p->mu);
      pthread_cond_broadcast(&p->cv_done);
      pthread_mutex_unlock(&p->mu);
    }
  }
}

static void* pool_worker(void* arg) {
  pool_t* p = (pool_t*)arg;
  uint64_t seen = 0;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    while (!p->stop && p->gen == seen) pthread_cond_wait(&p->cv, &p->mu);
    if (p->stop) {
      pthread_mutex_unlock(&p->mu);
      return NULL;
    }
    seen = p->gen;
    pthread_mutex_unlock(&p->mu);
    pool_run_chunks(p);
  }
}

static pool_t* pool_create(int lanes) {
  if (lanes <= 0) lanes = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (lanes < 1) lanes = 1;
  pool_t* p = (pool_t*)calloc(1, sizeof(pool_t));
  p->lanes = lanes;
  pthread_mutex_init(&p->mu, NULL);
  pthread_cond_init(&p->cv, NULL);
  pthread_cond_init(&p->cv_done, NULL);
  p->workers = (pthread_t*)calloc((size_t)lanes, sizeof(pthread_t));
  for (int i = 0; i < lanes - 1; ++i) pthread_create(&p->workers[i], NULL, pool_worker, p);
  return p;
}

static void pool_destroy(pool_t* p) {
  pthread_mutex_lock(&p->mu);
  p->stop = 1;
  pthread_cond_broadcast(&p->cv);
  pthread_mutex_unlock(&p->mu);
  for (int i = 0; i < p->lanes - 1; ++i) pthread_join(p->workers[i], NULL);
  free(p->workers);
  free(p);
}

static void parallel_for(pool_t* p, int64_t n, int64_t grain, chunk_fn fn, void* ctx) {
  if (n <= 0) return;
  const int64_t chunks = (n + grain - 1) / grain;
  if (chunks == 1 || p == NULL || p->lanes == 1) {
    for (int64_t c = 0; c < chunks; ++c) {
      int64_t b = c * grain;
      fn(ctx, b, b + grain < n ? b + grain : n);
    }
    return;
  }
  pthread_mutex_lock(&p->mu);
  p->fn = fn;
  p->ctx = ctx;
  p->n = n;
  p->grain = grain;
  p->chunks = chunks;
  p->next = 0;
  p->done = 0;
  p->gen++;
  pthread_cond_broadcast(&p->cv);
  pthread_mutex_unlock(&p->mu);
  pool_run_chunks(p);
  pthread_mutex_lock(&p->mu);
  while (__atomic_load_n(&p->done, __ATOMIC_ACQUIRE) < chunks) pthread_cond_wait(&p->cv_done, &p->mu);
  pthread_mutex_unlock(&p->mu);
}

/* ======================================================================
 * SimBatch standalone (sim_batch.hpp, dynamics.cpp:206-241)
 * ====================================================================== */
struct sgo_sim {
  sgo_robot m;
  int64_t n;
  real *q, *qd, *qt;
  sgo_pcg32* rng;
};

sgo_sim* sgo_sim_create(const sgo_robot* m, int64_t n, uint64_t seed, uint64_t salt) {
  sgo_sim* s = (sgo_sim*)calloc(1, sizeof(sgo_sim));
  s->m = *m;
  s->n = n;
  const int A = m->dof;
  s->q = (real*)calloc((size_t)(n * A), sizeof(real));
  s->qd = (real*)calloc((size_t)(n * A), sizeof(real));
  s->qt = (real*)calloc((size_t)(n * A), sizeof(real));
  s->rng = (sgo_pcg32*)calloc((size_t)n, sizeof(sgo_pcg32));
  double mid[SGO_MAX_JOINTS];
  mid_configuration(m, mid);
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < A; ++d) s->q[i * A + d] = s->qt[i * A + d] = (real)mid[d];
    sgo_make_stream(seed, salt * 0x100000000ULL + (uint64_t)i, &s->rng[i]);
  }
  return s;
}

void sgo_sim_destroy(sgo_sim* s) {
  if (!s) return;
  free(s->q);
  free(s->qd);
  free(s->qt);
  free(s->rng);
  free(s);
}

int sgo_sim_step(sgo_sim* s, const double* actions, const sgo_dyn* cfg, int64_t* saturated) {
  const int A = s->m.dof, jaw = sgo_jaw_dof(&s->m);
  int64_t sat = 0;
  int bad = 0;
  for (int64_t i = 0; i < s->n; ++i) {
    int r = dyn_row(&s->m, cfg, jaw, s->q + i * A, s->qd + i * A, s->qt + i * A, actions + i * A);
    if (r < 0) bad = 1;
    else sat += r;
  }
  if (saturated) *saturated = sat;
  return bad ? 1 : 0;
}

void sgo_sim_reset_rows(sgo_sim* s, const uint8_t* mask) { /* dynamics.cpp:206-223 */
  const int A = s->m.dof;
  for (int64_t i = 0; i < s->n; ++i) {
    if (!mask[i]) continue;
    for (int d = 0; d < A; ++d) {
      const sgo_joint* j = &s->m.joints[s->m.dof_to_joint[d]];
      const double quarter = 0.25 * (j->limit_hi - j->limit_lo);
      s->q[i * A + d] = (real)sgo_pcg32_uniform(&s->rng[i], j->limit_lo + quarter, j->limit_hi - quarter);
      s->qd[i * A + d] = 0;
      s->qt[i * A + d] = s->q[i * A + d];
    }
  }
}

void sgo_sim_get(const sgo_sim* s, double* q, double* qd, double* qt) {
  for (int64_t k = 0; k < s->n * s->m.dof; ++k) {
    if (q) q[k] = s->q[k];
    if (qd) qd[k] = s->qd[k];
    if (qt) qt[k] = s->qt[k];
  }
}

void sgo_sim_set(sgo_sim* s, const double* q, const double* qd, const double* qt) {
  for (int64_t k = 0; k < s->n * s->m.dof; ++k) {
    if (q) s->q[k] = (real)q[k];
    if (qd) s->qd[k] = (real)qd[k];
    if (qt) s->qt[k] = (real)qt[k];
  }
}

/* ======================================================================
 * Spline — spline.hpp:24-36, spline.cpp:28-72 (always fp64, like the device)
 * ====================================================================== */
#define SPLINE_SUBDIV 1000
#define DEGENERATE_LEN 1e-12

static void spline_eval(const double* c, double t0, double t, double* o) { /* spline.hpp:32-35 */
  const double u = t - t0;
  for (int k = 0; k < 3; ++k) o[k] = ((c[k] * u + c[3 + k]) * u + c[6 + k]) * u + c[9 + k];
}

static double norm3d(const double* a, const double* b) {
  double x = a[0] - b[0], y = a[1] - b[1], z = a[2] - b[2];
  return sqrt(x * x + y * y + z * z);
}

double sgo_spline_arc_length(const double* c, double t0, double t1, int subdivisions) {
  double total = 0.0, prev[3], p[3];
  spline_eval(c, t0, t0, prev);
  const double span = t1 - t0;
  for (int k = 1; k <= subdivisions; ++k) {
    spline_eval(c, t0, t0 + span * k / subdivisions, p);
    total += norm3d(p, prev);
    memcpy(prev, p, sizeof(p));
  }
  return total;
}

int sgo_spline_waypoints(const double* c, double t0, double t1, double spacing, double* out, int cap) {
  if (!(spacing > 0.0)) return -2;
  for (int k = 0; k < 12; ++k)
    if (!isfinite(c[k])) return -2;
  if (!isfinite(t0) || !isfinite(t1)) return -2;
  const double span = t1 - t0;
  static __thread double cum[SPLINE_SUBDIV + 1];
  static __thread double pts[SPLINE_SUBDIV + 1][3];
  cum[0] = 0.0;
  spline_eval(c, t0, t0, pts[0]);
  for (int k = 1; k <= SPLINE_SUBDIV; ++k) {
    spline_eval(c, t0, t0 + span * k / SPLINE_SUBDIV, pts[k]);
    cum[k] = cum[k - 1] + norm3d(pts[k], pts[k - 1]);
  }
  const double total = cum[SPLINE_SUBDIV];
  int count = 0;
#define PUSH(p)                                                   \
  do {                                                            \
    if (count < cap) memcpy(out + 3 * count, (p), 3 * sizeof(double)); \
    ++count;                                                      \
  } while (0)
  PUSH(pts[0]);
  if (total <= DEGENERATE_LEN) return count;
  int seg = 0;
  for (double s = spacing; s < total - DEGENERATE_LEN; s += spacing) {
    while (seg + 1 < SPLINE_SUBDIV && cum[seg + 1] < s) ++seg;
    const double seg_len = cum[seg + 1] - cum[seg];
    const double frac = seg_len > 0.0 ? (s - cum[seg]) / seg_len : 0.0;
    const double t = t0 + span * (seg + frac) / SPLINE_SUBDIV;
    double p[3];
    spline_eval(c, t0, t, p);
    PUSH(p);
  }
  PUSH(pts[SPLINE_SUBDIV]);
#undef PUSH
  return count;
}

/* ======================================================================
 * VecTaskEnv — envs.cpp (TargetReaching, PathFollowing; single tool)
 * ====================================================================== */
#define GOAL_REJECTION_LIMIT 1000 /* envs.cpp:29 */
#define ROW_GRAIN 256             /* envs.cpp:28, dynamics.cpp:25 */
#define WP_CAP 256

void sgo_env_cfg_default(sgo_env_cfg* c) { /* envs.hpp:42-63 */
  memset(c, 0, sizeof(*c));
  c->task = SGO_TARGET_REACHING;
  c->n_envs = 1024;
  c->episode_len = 300;
  c->goal_sigma = 0.05;
  c->goal_offset_clip = 0.2;
  c->reward_scale = -1.0;
  c->path_penalty = 1.0;
  c->success_radius = 0.005;
  c->success_hold = 10;
  c->workspace_radius = 0.0;
  c->waypoint_spacing = 0.02;
  c->tracking_vel_noise_std = 0.01;
  c->tracking_vel_clamp = 0.01;
  c->seed = 0;
  c->row_offset = 0;
  c->collision_threshold = 0.01;
  c->collision_penalty = 1.0;
  c->view_penalty = 0.1;
  c->render_w = 32; /* render.hpp:31-36 */
  c->render_h = 32;
  c->render_fov = 1.0471975511965976;
  c->render_near = 0.005;
  c->render_far = 2.0;
}

/* ======================================================================
 * Renderer — render.cpp:34-67 (Eigen formulas: toRotationMatrix, normalized()
 * = v / sqrt(squaredNorm), dot = (a0 b0 + a1 b1) + a2 b2)
 * ====================================================================== */
static void quat_to_rot_r(const real* q, real* R) { /* Quaternion::toRotationMatrix */
  const real tx = 2 * q[1], ty = 2 * q[2], tz = 2 * q[3];
  const real twx = tx * q[0], twy = ty * q[0], twz = tz * q[0];
  const real txx = tx * q[1], txy = ty * q[1], txz = tz * q[1];
  const real tyy = ty * q[2], tyz = tz * q[2], tzz = tz * q[3];
  R[0] = 1 - (tyy + tzz); R[1] = txy - twz; R[2] = txz + twy;
  R[3] = txy + twz; R[4] = 1 - (txx + tzz); R[5] = tyz - twx;
  R[6] = txz - twy; R[7] = tyz + twx; R[8] = 1 - (txx + tyy);
}

static void render_real(const real* pos, const real* quat, int w, int h, double fov, double near_,
                        double far_, const double* sph, int ns, real* out) {
  const real f = (real)(0.5 * w / tan(0.5 * fov)); /* focal length in pixels */
  real R[9];
  quat_to_rot_r(quat, R);
  for (int py = 0; py < h; ++py) {
    for (int px = 0; px < w; ++px) {
      const real u = (real)(px + 0.5 - 0.5 * w) / f;
      const real v = (real)(py + 0.5 - 0.5 * h) / f;
      const real dc[3] = {u, -v, -1}; /* top row looks up */
      real d[3];
      for (int r = 0; r < 3; ++r) d[r] = R[r * 3] * dc[0] + R[r * 3 + 1] * dc[1] + R[r * 3 + 2] * dc[2];
      const real nn = SGO_SQRT(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
      for (int r = 0; r < 3; ++r) d[r] = d[r] / nn;
      real best_t = (real)far_, value = 0;
      for (int s = 0; s < ns; ++s) {
        const double* S = sph + 5 * s;
        const real oc[3] = {pos[0] - (real)S[0], pos[1] - (real)S[1], pos[2] - (real)S[2]};
        const real rad = (real)S[3];
        const real b = oc[0] * d[0] + oc[1] * d[1] + oc[2] * d[2];
        const real disc = b * b - ((oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2]) - rad * rad);
        if (disc < 0) continue;
        const real t = -b - SGO_SQRT(disc);
        if (t < (real)near_ || t >= best_t) continue;
        best_t = t;
        real nrm[3];
        for (int k = 0; k < 3; ++k) nrm[k] = ((pos[k] + t * d[k]) - (real)S[k]) / rad;
        const real lambert = nrm[0] * -d[0] + nrm[1] * -d[1] + nrm[2] * -d[2];
        value = lambert > 0 ? (real)S[4] * lambert : 0;
      }
      out[py * w + px] = value;
    }
  }
}

void sgo_render(const double* cam_pos, const double* cam_quat, int w, int h, double fov, double near_,
                double far_, const double* spheres, int n_spheres, double* out) {
  real p[3], q[4];
  for (int k = 0; k < 3; ++k) p[k] = (real)cam_pos[k];
  for (int k = 0; k < 4; ++k) q[k] = (real)cam_quat[k];
  real* o = (real*)malloc(sizeof(real) * (size_t)(w * h));
  render_real(p, q, w, h, fov, near_, far_, spheres, n_spheres, o);
  for (int k = 0; k < w * h; ++k) out[k] = o[k];
  free(o);
}

struct sgo_env {
  sgo_env_cfg cfg;
  sgo_robot m;
  sgo_dyn dyn;
  int A, O, jaw;
  int64_t n;
  double center[3], radius;
  pool_t* pool;
  /* SimBatch */
  real *q, *qd, *qt;
  sgo_pcg32* rng;
  /* TaskState */
  real* goals;
  real *goal_spawn, *goal_vel; /* ActiveTracking (envs.cpp:199-201) */
  /* ImageMatching (envs.cpp:203-209): images n x wh, scenes n x 15, cameras n x 7 */
  int W, H, wh;
  real *timg, *cimg;
  double* scenes;
  real* tcam;
  int32_t *step_count, *hold_count, *wp_idx, *wp_len;
  int64_t* episode_count;
  real* wps; /* n x WP_CAP x 3 */
  /* tips & result */
  real* tips;
  real *obs, *tobs, *rewards, *task_error;
  uint8_t *terminated, *timed_out;
  int64_t saturations;
  int64_t goal_draws;
  /* per-chunk scratch */
  int64_t* chunk_sat;
  uint8_t* chunk_bad;
  uint8_t* chunk_bad_reward;
  const double* cur_actions;
  int err_code;
  char err[512];
};

/* envs.cpp:230-239 — components filled right-to-left (g++ argument order). */
static int sample_goal(sgo_env* e, sgo_pcg32* r, double* g) {
  const double s = e->cfg.goal_sigma;
  for (int attempt = 0; attempt < GOAL_REJECTION_LIMIT; ++attempt) {
    __atomic_fetch_add(&e->goal_draws, 1, __ATOMIC_RELAXED);
    double nz = 0.0 + s * sgo_pcg32_normal(r);
    double ny = 0.0 + s * sgo_pcg32_normal(r);
    double nx = 0.0 + s * sgo_pcg32_normal(r);
    g[0] = e->center[0] + nx;
    g[1] = e->center[1] + ny;
    g[2] = e->center[2] + nz;
    if (norm3d(g, e->center) <= e->radius) return 0;
  }
  return 2;
}

/* envs.cpp:241-267 */
static int sample_path(sgo_env* e, int64_t row) {
  sgo_pcg32* r = &e->rng[row];
  double c[12];
  for (int k = 0; k < 3; ++k) c[k] = sgo_pcg32_uniform(r, -0.5, 0.5);
  for (int k = 0; k < 3; ++k) c[3 + k] = sgo_pcg32_uniform(r, -0.5, 0.5);
  for (int k = 0; k < 3; ++k) c[6 + k] = sgo_pcg32_uniform(r, -0.3, 0.3);
  if (sample_goal(e, r, c + 9)) return 2;
  double max_off = 0.0, p[3];
  for (int k = 0; k <= 100; ++k) {
    spline_eval(c, 0.0, 0.01 * k, p);
    double d = norm3d(p, c + 9);
    max_off = max_off > d ? max_off : d; /* std::max(max_off, d) */
  }
  const double allowed = e->radius - norm3d(c + 9, e->center);
  if (max_off > 0.0 && max_off > allowed) {
    const double scale = 0.95 * (allowed > 0.0 ? allowed : 0.0) / max_off;
    for (int k = 0; k < 9; ++k) c[k] *= scale;
  }
  static __thread double w[WP_CAP * 3];
  int cnt = sgo_spline_waypoints(c, 0.0, 1.0, e->cfg.waypoint_spacing, w, WP_CAP);
  if (cnt < 0) return 2;
  if (cnt > WP_CAP) return 3;
  real* dst = e->wps + row * WP_CAP * 3;
  for (int k = 0; k < 3 * cnt; ++k) dst[k] = (real)w[k];
  e->wp_len[row] = cnt;
  e->wp_idx[row] = 0;
  return 0;
}

static void refresh_tip(sgo_env* e, int64_t row) { /* envs.cpp:297-302 */
  fk_r(&e->m, e->q + row * e->A, e->tips + row * 3, NULL);
}

/* envs.cpp:269-286: three spheres below the workspace, then a target view
 * from a mildly tilted configuration (sample_q_fraction 0.25, envs.cpp:31-39).
 * Eigen::Vector3d(x, y, z) arguments are drawn right to left (g++): z, y, x. */
static void sample_scene(sgo_env* e, int64_t row) {
  sgo_pcg32* r = &e->rng[row];
  const double s2 = 2.0 * e->cfg.goal_sigma;
  double* sc = e->scenes + row * 15;
  for (int k = 0; k < 3; ++k) {
    const double z = -(e->radius + sgo_pcg32_uniform(r, 0.1, 0.25));
    const double y = sgo_pcg32_uniform(r, -s2, s2);
    const double x = sgo_pcg32_uniform(r, -s2, s2);
    sc[5 * k + 0] = e->center[0] + x;
    sc[5 * k + 1] = e->center[1] + y;
    sc[5 * k + 2] = e->center[2] + z;
    sc[5 * k + 3] = sgo_pcg32_uniform(r, 0.02, 0.05);
    sc[5 * k + 4] = sgo_pcg32_uniform(r, 0.5, 1.0);
  }
  real q[SGO_MAX_JOINTS];
  for (int d = 0; d < e->A; ++d) {
    const sgo_joint* j = &e->m.joints[e->m.dof_to_joint[d]];
    const double margin = 0.5 * (1.0 - 0.25) * (j->limit_hi - j->limit_lo);
    q[d] = (real)sgo_pcg32_uniform(r, j->limit_lo + margin, j->limit_hi - margin);
  }
  real* cam = e->tcam + row * 7; /* identity tool base: compose is exact */
  fk_r(&e->m, q, cam, cam + 3);
  render_real(cam, cam + 3, e->W, e->H, e->cfg.render_fov, e->cfg.render_near, e->cfg.render_far, sc, 3,
              e->timg + row * e->wh);
}

static void render_row(sgo_env* e, int64_t row) { /* envs.cpp:288-295 */
  real cam[7];
  fk_r(&e->m, e->q + row * e->A, cam, cam + 3);
  render_real(cam, cam + 3, e->W, e->H, e->cfg.render_fov, e->cfg.render_near, e->cfg.render_far,
              e->scenes + row * 15, 3, e->cimg + row * e->wh);
}

static int reset_row(sgo_env* e, int64_t row) { /* envs.cpp:304-360 */
  const int A = e->A;
  sgo_pcg32* r = &e->rng[row];
  for (int d = 0; d < A; ++d) {
    const sgo_joint* j = &e->m.joints[e->m.dof_to_joint[d]];
    const double quarter = 0.25 * (j->limit_hi - j->limit_lo);
    e->q[row * A + d] = (real)sgo_pcg32_uniform(r, j->limit_lo + quarter, j->limit_hi - quarter);
    e->qd[row * A + d] = 0;
    e->qt[row * A + d] = e->q[row * A + d];
  }
  refresh_tip(e, row);
  if (e->cfg.task == SGO_TARGET_REACHING || e->cfg.task == SGO_ACTIVE_TRACKING) {
    double g[3];
    if (sample_goal(e, r, g)) return 2;
    for (int k = 0; k < 3; ++k) e->goals[row * 3 + k] = (real)g[k];
    if (e->cfg.task == SGO_ACTIVE_TRACKING) { /* envs.cpp:322-327 */
      for (int k = 0; k < 3; ++k) {
        e->goal_spawn[row * 3 + k] = (real)g[k];
        e->goal_vel[row * 3 + k] = 0;
      }
    }
  } else if (e->cfg.task == SGO_IMAGE_MATCHING) { /* envs.cpp:333-335 */
    sample_scene(e, row);
    render_row(e, row);
  } else { /* PathFollowing */
    int rc = sample_path(e, row);
    if (rc) return rc;
    for (int k = 0; k < 3; ++k) e->goals[row * 3 + k] = e->wps[row * WP_CAP * 3 + k];
  }
  e->step_count[row] = 0;
  e->hold_count[row] = 0;
  e->episode_count[row] += 1;
  return 0;
}

static void observe_row(sgo_env* e, int64_t row, real* dst) { /* envs.cpp:362-408 */
  const int A = e->A;
  real* out = dst + row * e->O;
  int off = 0;
  for (int d = 0; d < A; ++d) out[off++] = e->q[row * A + d];
  for (int d = 0; d < A; ++d) out[off++] = e->qd[row * A + d];
  for (int k = 0; k < 3; ++k) out[off++] = e->tips[row * 3 + k];
  for (int d = 0; d < A; ++d) out[off++] = e->qt[row * A + d];
  if (e->cfg.task == SGO_TARGET_REACHING || e->cfg.task == SGO_ACTIVE_TRACKING) {
    for (int k = 0; k < 3; ++k) out[off++] = e->goals[row * 3 + k];
  } else if (e->cfg.task == SGO_IMAGE_MATCHING) { /* envs.cpp:400-406 */
    for (int k = 0; k < e->wh; ++k) out[off++] = e->timg[row * e->wh + k];
    for (int k = 0; k < e->wh; ++k) out[off++] = e->cimg[row * e->wh + k];
  } else {
    const real* wp = e->wps + (row * WP_CAP + e->wp_idx[row]) * 3;
    for (int k = 0; k < 3; ++k) out[off++] = wp[k];
  }
}

static real dist3(const real* a, const real* b) {
  real x = a[0] - b[0], y = a[1] - b[1], z = a[2] - b[2];
  return SGO_SQRT(x * x + y * y + z * z);
}

static void phase_dynamics(void* ctx, int64_t b, int64_t end) { /* dynamics.cpp:124-188 */
  sgo_env* e = (sgo_env*)ctx;
  const int A = e->A;
  int64_t sat = 0;
  for (int64_t i = b; i < end; ++i) {
    int r = dyn_row(&e->m, &e->dyn, e->jaw, e->q + i * A, e->qd + i * A, e->qt + i * A,
                    e->cur_actions + i * A);
    if (r < 0) {
      e->chunk_bad[b / ROW_GRAIN] = 1;
      return;
    }
    sat += r;
  }
  e->chunk_sat[b / ROW_GRAIN] += sat;
}

static void phase_fk(void* ctx, int64_t b, int64_t end) { /* envs.cpp:456-463 */
  sgo_env* e = (sgo_env*)ctx;
  for (int64_t i = b; i < end; ++i) refresh_tip(e, i);
}

static void phase_render(void* ctx, int64_t b, int64_t end) { /* envs.cpp:464-473 */
  sgo_env* e = (sgo_env*)ctx;
  for (int64_t i = b; i < end; ++i) render_row(e, i);
}

static void phase_reward(void* ctx, int64_t b, int64_t end) { /* envs.cpp:478-594 */
  sgo_env* e = (sgo_env*)ctx;
  const real rho = (real)e->cfg.reward_scale, sr = (real)e->cfg.success_radius;
  for (int64_t i = b; i < end; ++i) {
    e->step_count[i] += 1;
    real reward = 0;
    int goal_met = 0;
    const real* tip = e->tips + i * 3;
    if (e->cfg.task == SGO_TARGET_REACHING) { /* envs.cpp:484-492 */
      const real dist = dist3(tip, e->goals + i * 3);
      reward = rho * dist;
      e->task_error[i] = dist;
      e->hold_count[i] = dist < sr ? e->hold_count[i] + 1 : 0;
      goal_met = e->hold_count[i] >= e->cfg.success_hold;
    } else if (e->cfg.task == SGO_ACTIVE_TRACKING) { /* envs.cpp:493-512 */
      real* g = e->goals + i * 3;
      const real dist = dist3(tip, g);
      reward = rho * dist;
      e->task_error[i] = dist;
      /* the goal drifts after the reward is scored */
      sgo_pcg32* r = &e->rng[i];
      real* vel = e->goal_vel + i * 3;
      const real* spawn = e->goal_spawn + i * 3;
      const real clip = (real)e->cfg.goal_offset_clip, vc = (real)e->cfg.tracking_vel_clamp;
      for (int k = 0; k < 3; ++k) g[k] += vel[k];
      for (int k = 0; k < 3; ++k) {
        const real lo = spawn[k] - clip, hi = spawn[k] + clip;
        g[k] = g[k] < lo ? lo : (hi < g[k] ? hi : g[k]); /* std::clamp */
        vel[k] += (real)(0.0 + e->cfg.tracking_vel_noise_std * sgo_pcg32_normal(r)); /* normal(0, std) */
        vel[k] = vel[k] < -vc ? -vc : (vc < vel[k] ? vc : vel[k]);
      }
    } else if (e->cfg.task == SGO_IMAGE_MATCHING) { /* envs.cpp:513-523 */
      const real* cur = e->cimg + i * e->wh;
      const real* tgt = e->timg + i * e->wh;
      real sum = 0;
      for (int k = 0; k < e->wh; ++k) sum += (real)fabs((double)(cur[k] - tgt[k]));
      const real err = sum / (real)e->wh;
      reward = -err;
      e->task_error[i] = err;
    } else { /* PathFollowing, envs.cpp:524-539 */
      const real* wps = e->wps + i * WP_CAP * 3;
      int32_t idx = e->wp_idx[i];
      const int32_t len = e->wp_len[i];
      const real dist = dist3(tip, wps + idx * 3);
      reward = -(real)e->cfg.path_penalty * dist;
      e->task_error[i] = dist;
      while (idx + 1 < len && dist3(tip, wps + idx * 3) < sr) ++idx;
      goal_met = idx + 1 == len && dist3(tip, wps + idx * 3) < sr;
      e->wp_idx[i] = idx;
      for (int k = 0; k < 3; ++k) e->goals[i * 3 + k] = wps[idx * 3 + k];
    }
    if (!isfinite((double)reward)) e->chunk_bad_reward[b / ROW_GRAIN] = 1;
    e->rewards[i] = reward;
    e->terminated[i] = goal_met ? 1 : 0;
    e->timed_out[i] = e->step_count[i] >= e->cfg.episode_len ? 1 : 0;
  }
}

static void phase_observe(void* ctx, int64_t b, int64_t end) { /* envs.cpp:410-423 */
  sgo_env* e = (sgo_env*)ctx;
  for (int64_t i = b; i < end; ++i) observe_row(e, i, e->obs);
}

static int env_fail(sgo_env* e, int code, const char* msg) {
  e->err_code = code;
  snprintf(e->err, sizeof(e->err), "%s", msg);
  return code;
}

sgo_env* sgo_env_create(const sgo_env_cfg* c, const sgo_robot* m, const sgo_dyn* dyn, int threads,
                        char* err, int errlen) {
  /* envs.cpp:65-81 (validate), 118-223 (ctor) */
  if (c->n_envs < 1) { seterr(err, errlen, "env.n_envs must be >= 1"); return NULL; }
  if (c->episode_len < 1) { seterr(err, errlen, "env.episode_len must be >= 1"); return NULL; }
  if (!(c->goal_sigma > 0.0)) { seterr(err, errlen, "env.goal_sigma must be > 0"); return NULL; }
  if (!(c->success_radius > 0.0)) { seterr(err, errlen, "env.success_radius must be > 0"); return NULL; }
  if (!(c->reward_scale < 0.0)) { seterr(err, errlen, "env.reward_scale (rho) must be < 0"); return NULL; }
  if (!(c->path_penalty > 0.0)) { seterr(err, errlen, "env.path_penalty (alpha) must be > 0"); return NULL; }
  if (c->success_hold < 1) { seterr(err, errlen, "env.success_hold must be >= 1"); return NULL; }
  if (!(c->waypoint_spacing > 0.0)) { seterr(err, errlen, "env.waypoint_spacing must be > 0"); return NULL; }
  if (c->workspace_radius < 0.0) { seterr(err, errlen, "env.workspace_radius must be >= 0"); return NULL; }
  if (c->tracking_vel_noise_std < 0.0) { seterr(err, errlen, "env.tracking_vel_noise_std must be >= 0"); return NULL; }
  if (!(c->tracking_vel_clamp > 0.0)) { seterr(err, errlen, "env.tracking_vel_clamp must be > 0"); return NULL; }
  if (c->task == SGO_IMAGE_MATCHING) { /* RenderConfig::validate (render.cpp:24-32) */
    if (c->render_w < 8 || c->render_h < 8) { seterr(err, errlen, "render: width and height must be >= 8"); return NULL; }
    if (!(c->render_near > 0.0) || !(c->render_near < c->render_far)) { seterr(err, errlen, "render: require 0 < near < far"); return NULL; }
    if (!(c->render_fov > 0.0) || !(c->render_fov < 3.1)) { seterr(err, errlen, "render: fov must be in (0, pi)"); return NULL; }
  }
  if (c->task != SGO_TARGET_REACHING && c->task != SGO_PATH_FOLLOWING && c->task != SGO_ACTIVE_TRACKING &&
      c->task != SGO_IMAGE_MATCHING) {
    seterr(err, errlen, "oracle: task %d not restated", c->task);
    return NULL;
  }
  sgo_env* e = (sgo_env*)calloc(1, sizeof(sgo_env));
  e->cfg = *c;
  e->m = *m;
  if (dyn) e->dyn = *dyn;
  else sgo_default_dynamics(m, &e->dyn);
  e->A = m->dof;
  e->O = 3 * m->dof + 6;
  if (c->task == SGO_IMAGE_MATCHING) { /* envs.cpp:185-188 */
    e->W = c->render_w;
    e->H = c->render_h;
    e->wh = e->W * e->H;
    e->O = 3 * m->dof + 3 + 2 * e->wh;
  }
  e->jaw = sgo_jaw_dof(m);
  e->n = c->n_envs;
  e->radius = c->workspace_radius > 0.0 ? c->workspace_radius : 3.0 * c->goal_sigma; /* :134 */
  double mid[SGO_MAX_JOINTS], tq[4];
  mid_configuration(m, mid);
  fk_d(m, mid, e->center, tq); /* envs.cpp:161-162 (identity tool base) */
  e->pool = threads == 1 ? NULL : pool_create(threads);
  const int64_t n = e->n, A = e->A, O = e->O;
  e->q = (real*)calloc((size_t)(n * A), sizeof(real));
  e->qd = (real*)calloc((size_t)(n * A), sizeof(real));
  e->qt = (real*)calloc((size_t)(n * A), sizeof(real));
  e->rng = (sgo_pcg32*)calloc((size_t)n, sizeof(sgo_pcg32));
  for (int64_t i = 0; i < n; ++i) { /* dynamics.cpp:225-241, salt 0 */
    for (int d = 0; d < A; ++d) e->q[i * A + d] = e->qt[i * A + d] = (real)mid[d];
    sgo_make_stream(c->seed, (uint64_t)(c->row_offset + i), &e->rng[i]);
  }
  e->goals = (real*)calloc((size_t)(n * 3), sizeof(real));
  e->step_count = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  e->hold_count = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  e->wp_idx = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  e->wp_len = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  e->episode_count = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  if (c->task == SGO_PATH_FOLLOWING) e->wps = (real*)calloc((size_t)(n * WP_CAP * 3), sizeof(real));
  if (c->task == SGO_IMAGE_MATCHING) {
    e->timg = (real*)calloc((size_t)(n * e->wh), sizeof(real));
    e->cimg = (real*)calloc((size_t)(n * e->wh), sizeof(real));
    e->scenes = (double*)calloc((size_t)(n * 15), sizeof(double));
    e->tcam = (real*)calloc((size_t)(n * 7), sizeof(real));
  }
  if (c->task == SGO_ACTIVE_TRACKING) {
    e->goal_spawn = (real*)calloc((size_t)(n * 3), sizeof(real));
    e->goal_vel = (real*)calloc((size_t)(n * 3), sizeof(real));
  }
  e->tips = (real*)calloc((size_t)(n * 3), sizeof(real));
  e->obs = (real*)calloc((size_t)(n * O), sizeof(real));
  e->tobs = (real*)calloc((size_t)(n * O), sizeof(real));
  e->rewards = (real*)calloc((size_t)n, sizeof(real));
  e->task_error = (real*)calloc((size_t)n, sizeof(real));
  e->terminated = (uint8_t*)calloc((size_t)n, 1);
  e->timed_out = (uint8_t*)calloc((size_t)n, 1);
  const int64_t chunks = (n + ROW_GRAIN - 1) / ROW_GRAIN;
  e->chunk_sat = (int64_t*)calloc((size_t)chunks, sizeof(int64_t));
  e->chunk_bad = (uint8_t*)calloc((size_t)chunks, 1);
  e->chunk_bad_reward = (uint8_t*)calloc((size_t)chunks, 1);
  return e;
}

void sgo_env_destroy(sgo_env* e) {
  if (!e) return;
  if (e->pool) pool_destroy(e->pool);
  free(e->q); free(e->qd); free(e->qt); free(e->rng); free(e->goals);
  free(e->goal_spawn); free(e->goal_vel);
  free(e->timg); free(e->cimg); free(e->scenes); free(e->tcam);
  free(e->step_count); free(e->hold_count); free(e->wp_idx); free(e->wp_len);
  free(e->episode_count); free(e->wps); free(e->tips); free(e->obs); free(e->tobs);
  free(e->rewards); free(e->task_error); free(e->terminated); free(e->timed_out);
  free(e->chunk_sat); free(e->chunk_bad); free(e->chunk_bad_reward);
  free(e);
}

int sgo_env_obs_dim(const sgo_env* e) { return e->O; }
int sgo_env_action_dim(const sgo_env* e) { return e->A; }
int sgo_env_lanes(const sgo_env* e) { return e->pool ? e->pool->lanes : 1; }
const char* sgo_env_error(const sgo_env* e) { return e->err; }

int sgo_env_reset(sgo_env* e) { /* envs.cpp:425-435 */
  for (int64_t i = 0; i < e->n; ++i) {
    int rc = reset_row(e, i);
    if (rc == 3) return env_fail(e, 1, "waypoint table capacity exceeded");
    if (rc) return env_fail(e, 2, "goal sampling rejected 1000 candidates; workspace_radius is misconfigured for goal_sigma");
    e->episode_count[i] = 0;
  }
  parallel_for(e->pool, e->n, ROW_GRAIN, phase_observe, e);
  memset(e->terminated, 0, (size_t)e->n);
  memset(e->timed_out, 0, (size_t)e->n);
  for (int64_t i = 0; i < e->n; ++i) e->rewards[i] = 0;
  return 0;
}

int sgo_env_step(sgo_env* e, const double* actions) { /* envs.cpp:437-617 */
  const int64_t n = e->n, chunks = (n + ROW_GRAIN - 1) / ROW_GRAIN;
  memset(e->chunk_sat, 0, (size_t)chunks * sizeof(int64_t));
  memset(e->chunk_bad, 0, (size_t)chunks);
  memset(e->chunk_bad_reward, 0, (size_t)chunks);
  e->cur_actions = actions;
  parallel_for(e->pool, n, ROW_GRAIN, phase_dynamics, e);
  e->saturations = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    if (e->chunk_bad[c]) return env_fail(e, 1, "dynamics.step: non-finite action entry");
  }
  for (int64_t c = 0; c < chunks; ++c) e->saturations += e->chunk_sat[c];
  parallel_for(e->pool, n, ROW_GRAIN, phase_fk, e);
  if (e->cfg.task == SGO_IMAGE_MATCHING) parallel_for(e->pool, n, ROW_GRAIN, phase_render, e);
  parallel_for(e->pool, n, ROW_GRAIN, phase_reward, e);
  for (int64_t c = 0; c < chunks; ++c)
    if (e->chunk_bad_reward[c]) return env_fail(e, 1, "env.step: non-finite reward");
  parallel_for(e->pool, n, ROW_GRAIN, phase_observe, e);
  const int O = e->O;
  int any = 0;
  for (int64_t i = 0; i < n; ++i) { /* envs.cpp:605-611 (serial scan) */
    if (e->terminated[i] || e->timed_out[i]) {
      memcpy(e->tobs + i * O, e->obs + i * O, (size_t)O * sizeof(real));
      any = 1;
    }
  }
  if (any) { /* envs.cpp:612-615 (serial resets, then re-observe) */
    for (int64_t i = 0; i < n; ++i) {
      if (e->terminated[i] || e->timed_out[i]) {
        int rc = reset_row(e, i);
        if (rc == 3) return env_fail(e, 1, "waypoint table capacity exceeded");
        if (rc) return env_fail(e, 2, "goal sampling rejected 1000 candidates; workspace_radius is misconfigured for goal_sigma");
      }
    }
    for (int64_t i = 0; i < n; ++i)
      if (e->terminated[i] || e->timed_out[i]) observe_row(e, i, e->obs);
  }
  return 0;
}

void sgo_env_get_obs(const sgo_env* e, double* obs, double* tobs) {
  for (int64_t k = 0; k < e->n * e->O; ++k) {
    if (obs) obs[k] = e->obs[k];
    if (tobs) tobs[k] = e->tobs[k];
  }
}

void sgo_env_get_result(const sgo_env* e, double* rewards, uint8_t* term, uint8_t* tout,
                        double* task_error, int64_t* sat) {
  for (int64_t i = 0; i < e->n; ++i) {
    if (rewards) rewards[i] = e->rewards[i];
    if (term) term[i] = e->terminated[i];
    if (tout) tout[i] = e->timed_out[i];
    if (task_error) task_error[i] = e->task_error[i];
  }
  if (sat) *sat = e->saturations;
}

void sgo_env_get_state(const sgo_env* e, double* q, double* qd, double* qt, double* tips,
                       double* goals) {
  for (int64_t k = 0; k < e->n * e->A; ++k) {
    if (q) q[k] = e->q[k];
    if (qd) qd[k] = e->qd[k];
    if (qt) qt[k] = e->qt[k];
  }
  for (int64_t k = 0; k < e->n * 3; ++k) {
    if (tips) tips[k] = e->tips[k];
    if (goals) goals[k] = e->goals[k];
  }
}

void sgo_env_get_counters(const sgo_env* e, int32_t* sc, int32_t* hc, int64_t* ec, int32_t* wi,
                          int32_t* wl) {
  for (int64_t i = 0; i < e->n; ++i) {
    if (sc) sc[i] = e->step_count[i];
    if (hc) hc[i] = e->hold_count[i];
    if (ec) ec[i] = e->episode_count[i];
    if (wi) wi[i] = e->wp_idx[i];
    if (wl) wl[i] = e->wp_len[i];
  }
}

void sgo_env_get_rng(const sgo_env* e, uint64_t* state, uint64_t* inc) {
  for (int64_t i = 0; i < e->n; ++i) {
    if (state) state[i] = e->rng[i].state;
    if (inc) inc[i] = e->rng[i].inc;
  }
}

int sgo_env_get_waypoints(const sgo_env* e, int64_t row, double* out, int cap) {
  if (!e->wps) return 0;
  int cnt = e->wp_len[row];
  for (int k = 0; k < cnt && k < cap; ++k)
    for (int c = 0; c < 3; ++c) out[k * 3 + c] = e->wps[(row * WP_CAP + k) * 3 + c];
  return cnt;
}

void sgo_env_get_images(const sgo_env* e, double* target, double* current, double* scenes,
                        double* tcams) {
  if (!e->timg) return;
  for (int64_t k = 0; k < e->n * e->wh; ++k) {
    if (target) target[k] = e->timg[k];
    if (current) current[k] = e->cimg[k];
  }
  for (int64_t k = 0; k < e->n * 15; ++k)
    if (scenes) scenes[k] = e->scenes[k];
  for (int64_t k = 0; k < e->n * 7; ++k)
    if (tcams) tcams[k] = e->tcam[k];
}

void sgo_env_workspace(const sgo_env* e, double* center, double* radius) {
  for (int k = 0; k < 3; ++k) center[k] = e->center[k];
  *radius = e->radius;
}

int64_t sgo_env_goal_draws(const sgo_env* e) { return e->goal_draws; }

void sgo_env_set_state(sgo_env* e, const double* q, const double* qd, const double* qt) {
  for (int64_t k = 0; k < e->n * e->A; ++k) {
    if (q) e->q[k] = (real)q[k];
    if (qd) e->qd[k] = (real)qd[k];
    if (qt) e->qt[k] = (real)qt[k];
  }
}

/* ======================================================================
 * MultiToolReaching — envs.cpp:90-116, 118-223, 304-360, 362-408, 437-617
 * (one SimBatch per tool; tool-major action / observation columns)
 * ====================================================================== */
double sgo_multi_tool_min_separation(const double* tips, int n) { /* envs.cpp:90-99 */
  double best = INFINITY;
  if (n < 2) return best;
  for (int i = 0; i + 1 < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double d = norm3d(tips + 3 * i, tips + 3 * j);
      best = d < best ? d : best; /* std::min(best, d) */
    }
  return best;
}

void sgo_default_tool_bases(int n_tools, double r, sgo_pose* b) { /* envs.cpp:101-116 */
  for (int t = 0; t < n_tools; ++t) {
    memset(&b[t], 0, sizeof(b[t]));
    b[t].quat[0] = 1.0;
  }
  if (n_tools == 1) return;
  const double dx = 0.7 * r;
  b[0].xyz[0] = -dx;
  b[1].xyz[0] = dx;
  if (n_tools >= 3) { /* camera arm behind the scene, pitched toward it */
    b[2].xyz[1] = -2.0 * r;
    b[2].xyz[2] = 0.5 * r;
    quat_from_rpy(0.9, 0.0, 0.0, b[2].quat);
  }
  for (int t = 3; t < n_tools; ++t) b[t].xyz[1] = ((double)t - 1.0) * 2.0 * dx;
}

struct sgo_mt_env {
  sgo_env_cfg cfg;
  int T, A, O;
  int64_t n;
  sgo_robot m[SGO_MAX_TOOLS];
  sgo_dyn dyn[SGO_MAX_TOOLS];
  int dof[SGO_MAX_TOOLS], off[SGO_MAX_TOOLS], jaw[SGO_MAX_TOOLS], ecm[SGO_MAX_TOOLS];
  sgo_pose base[SGO_MAX_TOOLS];
  double center[SGO_MAX_TOOLS][3], radius;
  pool_t* pool;
  real *q[SGO_MAX_TOOLS], *qd[SGO_MAX_TOOLS], *qt[SGO_MAX_TOOLS]; /* n x dof_t */
  sgo_pcg32* rng[SGO_MAX_TOOLS];
  real *tips, *tquat; /* n x T x 3, n x T x 4 (world frame) */
  real* goals;        /* n x 3T */
  int32_t *step_count, *hold_count;
  int64_t* episode_count;
  real *obs, *tobs, *rewards, *task_error;
  uint8_t *terminated, *timed_out;
  int64_t saturations;
  int64_t* chunk_sat;
  uint8_t *chunk_bad, *chunk_bad_reward;
  const double* cur_actions;
  char err[512];
};

/* tip_pose / refresh_tips (envs.cpp:225-228, 297-302): base ∘ FK */
static void mt_refresh_tips(struct sgo_mt_env* e, int64_t row) {
  for (int t = 0; t < e->T; ++t) {
    real p[3], qq[4], bp[3], bq[4], v[3];
    fk_r(&e->m[t], e->q[t] + row * e->dof[t], p, qq);
    for (int k = 0; k < 3; ++k) bp[k] = (real)e->base[t].xyz[k];
    for (int k = 0; k < 4; ++k) bq[k] = (real)e->base[t].quat[k];
    qrot_r(bq, p, v); /* Pose::compose: position + orientation * other.position */
    real* tp = e->tips + (row * e->T + t) * 3;
    for (int k = 0; k < 3; ++k) tp[k] = bp[k] + v[k];
    qmul_r(bq, qq, e->tquat + (row * e->T + t) * 4);
  }
}

/* Camera arm goal: midpoint of the other tools' tips (envs.cpp:339-348, 547-555). */
static void mt_camera_mid(const struct sgo_mt_env* e, int64_t row, int t, real* mid) {
  mid[0] = mid[1] = mid[2] = 0;
  int count = 0;
  for (int u = 0; u < e->T; ++u) {
    if (u == t) continue;
    const real* tp = e->tips + (row * e->T + u) * 3;
    for (int k = 0; k < 3; ++k) mid[k] += tp[k];
    ++count;
  }
  for (int k = 0; k < 3; ++k) mid[k] /= (real)count;
}

static int mt_sample_goal(const struct sgo_mt_env* e, sgo_pcg32* r, const double* c, double* g) {
  const double s = e->cfg.goal_sigma; /* envs.cpp:230-239, z drawn first (g++) */
  for (int attempt = 0; attempt < GOAL_REJECTION_LIMIT; ++attempt) {
    double nz = 0.0 + s * sgo_pcg32_normal(r);
    double ny = 0.0 + s * sgo_pcg32_normal(r);
    double nx = 0.0 + s * sgo_pcg32_normal(r);
    g[0] = c[0] + nx;
    g[1] = c[1] + ny;
    g[2] = c[2] + nz;
    if (norm3d(g, c) <= e->radius) return 0;
  }
  return 2;
}

static int mt_reset_row(struct sgo_mt_env* e, int64_t row) { /* envs.cpp:304-360 */
  for (int t = 0; t < e->T; ++t) {
    const int A = e->dof[t];
    sgo_pcg32* r = &e->rng[t][row];
    for (int d = 0; d < A; ++d) {
      const sgo_joint* j = &e->m[t].joints[e->m[t].dof_to_joint[d]];
      const double quarter = 0.25 * (j->limit_hi - j->limit_lo);
      e->q[t][row * A + d] = (real)sgo_pcg32_uniform(r, j->limit_lo + quarter, j->limit_hi - quarter);
      e->qd[t][row * A + d] = 0;
      e->qt[t][row * A + d] = e->q[t][row * A + d];
    }
  }
  mt_refresh_tips(e, row);
  for (int t = 0; t < e->T; ++t) { /* envs.cpp:336-354 */
    real* g = e->goals + row * 3 * e->T + 3 * t;
    if (e->ecm[t]) {
      mt_camera_mid(e, row, t, g);
    } else {
      double gd[3];
      if (mt_sample_goal(e, &e->rng[t][row], e->center[t], gd)) return 2;
      for (int k = 0; k < 3; ++k) g[k] = (real)gd[k];
    }
  }
  e->step_count[row] = 0;
  e->hold_count[row] = 0;
  e->episode_count[row] += 1;
  return 0;
}

static void mt_observe_row(struct sgo_mt_env* e, int64_t row, real* dst) { /* envs.cpp:362-408 */
  real* out = dst + row * e->O;
  int off = 0;
  for (int t = 0; t < e->T; ++t)
    for (int d = 0; d < e->dof[t]; ++d) out[off++] = e->q[t][row * e->dof[t] + d];
  for (int t = 0; t < e->T; ++t)
    for (int d = 0; d < e->dof[t]; ++d) out[off++] = e->qd[t][row * e->dof[t] + d];
  for (int t = 0; t < e->T; ++t)
    for (int k = 0; k < 3; ++k) out[off++] = e->tips[(row * e->T + t) * 3 + k];
  for (int t = 0; t < e->T; ++t)
    for (int d = 0; d < e->dof[t]; ++d) out[off++] = e->qt[t][row * e->dof[t] + d];
  for (int k = 0; k < 3 * e->T; ++k) out[off++] = e->goals[row * 3 * e->T + k];
}

static void mt_phase_dynamics(void* ctx, int64_t b, int64_t end) { /* dynamics.cpp:124-188 per tool */
  struct sgo_mt_env* e = (struct sgo_mt_env*)ctx;
  int64_t sat = 0;
  for (int64_t i = b; i < end; ++i) {
    for (int t = 0; t < e->T; ++t) {
      const int A = e->dof[t];
      int r = dyn_row(&e->m[t], &e->dyn[t], e->jaw[t], e->q[t] + i * A, e->qd[t] + i * A,
                      e->qt[t] + i * A, e->cur_actions + i * e->A + e->off[t]);
      if (r < 0) {
        e->chunk_bad[b / ROW_GRAIN] = 1;
        return;
      }
      sat += r;
    }
  }
  e->chunk_sat[b / ROW_GRAIN] += sat;
}

static void mt_phase_fk(void* ctx, int64_t b, int64_t end) { /* envs.cpp:456-463 */
  struct sgo_mt_env* e = (struct sgo_mt_env*)ctx;
  for (int64_t i = b; i < end; ++i) mt_refresh_tips(e, i);
}

static void mt_phase_reward(void* ctx, int64_t b, int64_t end) { /* envs.cpp:540-593 */
  struct sgo_mt_env* e = (struct sgo_mt_env*)ctx;
  const int T = e->T;
  const real rho = (real)e->cfg.reward_scale, sr = (real)e->cfg.success_radius;
  for (int64_t i = b; i < end; ++i) {
    e->step_count[i] += 1;
    real reward = 0, err_sum = 0;
    int err_count = 0, all_in = 1;
    const real* tips = e->tips + i * T * 3;
    real* goals = e->goals + i * 3 * T;
    for (int t = 0; t < T; ++t) {
      const real* tp = tips + 3 * t;
      if (e->ecm[t]) {
        real mid[3];
        mt_camera_mid(e, i, t, mid);
        for (int k = 0; k < 3; ++k) goals[3 * t + k] = mid[k];
        const real down[3] = {0, 0, -1};
        real axis[3];
        qrot_r(e->tquat + (i * T + t) * 4, down, axis);
        const real to_mid[3] = {mid[0] - tp[0], mid[1] - tp[1], mid[2] - tp[2]};
        const real nrm = SGO_SQRT(to_mid[0] * to_mid[0] + to_mid[1] * to_mid[1] + to_mid[2] * to_mid[2]);
        if (nrm > (real)1e-12) {
          /* Eigen normalized(): v / norm */
          real c = axis[0] * (to_mid[0] / nrm) + axis[1] * (to_mid[1] / nrm) + axis[2] * (to_mid[2] / nrm);
          c = c < (real)-1 ? (real)-1 : ((real)1 < c ? (real)1 : c); /* std::clamp */
          reward += -(real)e->cfg.view_penalty * SGO_ACOS(c);
        }
      } else {
        const real dist = dist3(tp, goals + 3 * t);
        reward += rho * dist;
        err_sum += dist;
        ++err_count;
        if (dist >= sr) all_in = 0;
      }
    }
    real min_sep = (real)INFINITY;
    for (int t = 0; t + 1 < T; ++t)
      for (int u = t + 1; u < T; ++u) {
        const real d = dist3(tips + 3 * t, tips + 3 * u);
        min_sep = d < min_sep ? d : min_sep;
      }
    if (min_sep < (real)e->cfg.collision_threshold) reward += -(real)e->cfg.collision_penalty;
    e->task_error[i] = err_count > 0 ? err_sum / (real)err_count : 0;
    e->hold_count[i] = all_in ? e->hold_count[i] + 1 : 0;
    const int goal_met = e->hold_count[i] >= e->cfg.success_hold;
    if (!isfinite((double)reward)) e->chunk_bad_reward[b / ROW_GRAIN] = 1;
    e->rewards[i] = reward;
    e->terminated[i] = goal_met ? 1 : 0;
    e->timed_out[i] = e->step_count[i] >= e->cfg.episode_len ? 1 : 0;
  }
}

static void mt_phase_observe(void* ctx, int64_t b, int64_t end) {
  struct sgo_mt_env* e = (struct sgo_mt_env*)ctx;
  for (int64_t i = b; i < end; ++i) mt_observe_row(e, i, e->obs);
}

sgo_mt_env* sgo_mt_env_create(const sgo_env_cfg* c, const sgo_robot* models, int n_tools,
                              const sgo_pose* bases, const sgo_dyn* dyn, int threads, char* err,
                              int errlen) {
  if (c->n_envs < 1) { seterr(err, errlen, "env.n_envs must be >= 1"); return NULL; }
  if (c->episode_len < 1) { seterr(err, errlen, "env.episode_len must be >= 1"); return NULL; }
  if (!(c->goal_sigma > 0.0)) { seterr(err, errlen, "env.goal_sigma must be > 0"); return NULL; }
  if (!(c->success_radius > 0.0)) { seterr(err, errlen, "env.success_radius must be > 0"); return NULL; }
  if (!(c->reward_scale < 0.0)) { seterr(err, errlen, "env.reward_scale (rho) must be < 0"); return NULL; }
  if (c->success_hold < 1) { seterr(err, errlen, "env.success_hold must be >= 1"); return NULL; }
  if (c->workspace_radius < 0.0) { seterr(err, errlen, "env.workspace_radius must be >= 0"); return NULL; }
  if (c->collision_threshold < 0.0) { seterr(err, errlen, "env.collision_threshold must be >= 0"); return NULL; }
  if (c->collision_penalty < 0.0) { seterr(err, errlen, "env.collision_penalty must be >= 0"); return NULL; }
  if (c->view_penalty < 0.0) { seterr(err, errlen, "env.view_penalty must be >= 0"); return NULL; }
  if (n_tools < 2) { seterr(err, errlen, "multi_tool_reaching requires >= 2 robots"); return NULL; }
  if (n_tools > SGO_MAX_TOOLS) { seterr(err, errlen, "oracle: at most %d tools", SGO_MAX_TOOLS); return NULL; }
  struct sgo_mt_env* e = (struct sgo_mt_env*)calloc(1, sizeof(*e));
  e->cfg = *c;
  e->T = n_tools;
  e->n = c->n_envs;
  e->radius = c->workspace_radius > 0.0 ? c->workspace_radius : 3.0 * c->goal_sigma; /* :134 */
  if (bases) memcpy(e->base, bases, sizeof(sgo_pose) * (size_t)n_tools);
  else sgo_default_tool_bases(n_tools, e->radius, e->base);
  const int64_t n = e->n;
  for (int t = 0; t < n_tools; ++t) {
    e->m[t] = models[t];
    if (dyn) e->dyn[t] = dyn[t];
    else sgo_default_dynamics(&models[t], &e->dyn[t]);
    e->dof[t] = models[t].dof;
    e->off[t] = e->A;
    e->jaw[t] = sgo_jaw_dof(&models[t]);
    e->ecm[t] = strcmp(models[t].name, "ecm") == 0; /* models_[t].name == "ecm" */
    e->A += models[t].dof;
    /* workspace centre: base.transform_point(FK(mid).position) (envs.cpp:159-161) */
    double mid[SGO_MAX_JOINTS], p[3], tq[4], v[3];
    mid_configuration(&models[t], mid);
    fk_d(&models[t], mid, p, tq);
    qrot_d(e->base[t].quat, p, v);
    for (int k = 0; k < 3; ++k) e->center[t][k] = e->base[t].xyz[k] + v[k];
    const int A = e->dof[t];
    e->q[t] = (real*)calloc((size_t)(n * A), sizeof(real));
    e->qd[t] = (real*)calloc((size_t)(n * A), sizeof(real));
    e->qt[t] = (real*)calloc((size_t)(n * A), sizeof(real));
    e->rng[t] = (sgo_pcg32*)calloc((size_t)n, sizeof(sgo_pcg32));
    for (int64_t i = 0; i < n; ++i) { /* SimBatch::create, salt = tool (dynamics.cpp:225-241) */
      for (int d = 0; d < A; ++d) e->q[t][i * A + d] = e->qt[t][i * A + d] = (real)mid[d];
      sgo_make_stream(c->seed, ((uint64_t)t << 32) + (uint64_t)(c->row_offset + i), &e->rng[t][i]);
    }
  }
  e->O = 3 * e->A + 6 * n_tools; /* envs.cpp:166-192 */
  e->pool = threads == 1 ? NULL : pool_create(threads);
  e->tips = (real*)calloc((size_t)(n * n_tools * 3), sizeof(real));
  e->tquat = (real*)calloc((size_t)(n * n_tools * 4), sizeof(real));
  e->goals = (real*)calloc((size_t)(n * n_tools * 3), sizeof(real));
  e->step_count = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  e->hold_count = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  e->episode_count = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  e->obs = (real*)calloc((size_t)(n * e->O), sizeof(real));
  e->tobs = (real*)calloc((size_t)(n * e->O), sizeof(real));
  e->rewards = (real*)calloc((size_t)n, sizeof(real));
  e->task_error = (real*)calloc((size_t)n, sizeof(real));
  e->terminated = (uint8_t*)calloc((size_t)n, 1);
  e->timed_out = (uint8_t*)calloc((size_t)n, 1);
  const int64_t chunks = (n + ROW_GRAIN - 1) / ROW_GRAIN;
  e->chunk_sat = (int64_t*)calloc((size_t)chunks, sizeof(int64_t));
  e->chunk_bad = (uint8_t*)calloc((size_t)chunks, 1);
  e->chunk_bad_reward = (uint8_t*)calloc((size_t)chunks, 1);
  return e;
}

void sgo_mt_env_destroy(sgo_mt_env* e) {
  if (!e) return;
  if (e->pool) pool_destroy(e->pool);
  for (int t = 0; t < e->T; ++t) {
    free(e->q[t]); free(e->qd[t]); free(e->qt[t]); free(e->rng[t]);
  }
  free(e->tips); free(e->tquat); free(e->goals); free(e->step_count); free(e->hold_count);
  free(e->episode_count); free(e->obs); free(e->tobs); free(e->rewards); free(e->task_error);
  free(e->terminated); free(e->timed_out); free(e->chunk_sat); free(e->chunk_bad);
  free(e->chunk_bad_reward);
  free(e);
}

void sgo_mt_env_dims(const sgo_mt_env* e, int* action_dim, int* obs_dim, int* dofs) {
  if (action_dim) *action_dim = e->A;
  if (obs_dim) *obs_dim = e->O;
  if (dofs)
    for (int t = 0; t < e->T; ++t) dofs[t] = e->dof[t];
}

const char* sgo_mt_env_error(const sgo_mt_env* e) { return e->err; }

static int mt_fail(sgo_mt_env* e, int code, const char* msg) {
  snprintf(e->err, sizeof(e->err), "%s", msg);
  return code;
}

int sgo_mt_env_reset(sgo_mt_env* e) { /* envs.cpp:425-435 */
  for (int64_t i = 0; i < e->n; ++i) {
    if (mt_reset_row(e, i))
      return mt_fail(e, 2, "goal sampling rejected 1000 candidates; workspace_radius is misconfigured for goal_sigma");
    e->episode_count[i] = 0;
  }
  parallel_for(e->pool, e->n, ROW_GRAIN, mt_phase_observe, e);
  memset(e->terminated, 0, (size_t)e->n);
  memset(e->timed_out, 0, (size_t)e->n);
  for (int64_t i = 0; i < e->n; ++i) e->rewards[i] = 0;
  return 0;
}

int sgo_mt_env_step(sgo_mt_env* e, const double* actions) { /* envs.cpp:437-617 */
  const int64_t n = e->n, chunks = (n + ROW_GRAIN - 1) / ROW_GRAIN;
  memset(e->chunk_sat, 0, (size_t)chunks * sizeof(int64_t));
  memset(e->chunk_bad, 0, (size_t)chunks);
  memset(e->chunk_bad_reward, 0, (size_t)chunks);
  e->cur_actions = actions;
  parallel_for(e->pool, n, ROW_GRAIN, mt_phase_dynamics, e);
  e->saturations = 0;
  for (int64_t c = 0; c < chunks; ++c)
    if (e->chunk_bad[c]) return mt_fail(e, 1, "dynamics.step: non-finite action entry");
  for (int64_t c = 0; c < chunks; ++c) e->saturations += e->chunk_sat[c];
  parallel_for(e->pool, n, ROW_GRAIN, mt_phase_fk, e);
  parallel_for(e->pool, n, ROW_GRAIN, mt_phase_reward, e);
  for (int64_t c = 0; c < chunks; ++c)
    if (e->chunk_bad_reward[c]) return mt_fail(e, 1, "env.step: non-finite reward");
  parallel_for(e->pool, n, ROW_GRAIN, mt_phase_observe, e);
  const int O = e->O;
  int any = 0;
  for (int64_t i = 0; i < n; ++i)
    if (e->terminated[i] || e->timed_out[i]) {
      memcpy(e->tobs + i * O, e->obs + i * O, (size_t)O * sizeof(real));
      any = 1;
    }
  if (any) {
    for (int64_t i = 0; i < n; ++i)
      if ((e->terminated[i] || e->timed_out[i]) && mt_reset_row(e, i))
        return mt_fail(e, 2, "goal sampling rejected 1000 candidates; workspace_radius is misconfigured for goal_sigma");
    for (int64_t i = 0; i < n; ++i)
      if (e->terminated[i] || e->timed_out[i]) mt_observe_row(e, i, e->obs);
  }
  return 0;
}

void sgo_mt_env_get_obs(const sgo_mt_env* e, double* obs, double* tobs) {
  for (int64_t k = 0; k < e->n * e->O; ++k) {
    if (obs) obs[k] = e->obs[k];
    if (tobs) tobs[k] = e->tobs[k];
  }
}

void sgo_mt_env_get_result(const sgo_mt_env* e, double* rewards, uint8_t* term, uint8_t* tout,
                           double* task_error, int64_t* sat) {
  for (int64_t i = 0; i < e->n; ++i) {
    if (rewards) rewards[i] = e->rewards[i];
    if (term) term[i] = e->terminated[i];
    if (tout) tout[i] = e->timed_out[i];
    if (task_error) task_error[i] = e->task_error[i];
  }
  if (sat) *sat = e->saturations;
}

void sgo_mt_env_get_state(const sgo_mt_env* e, double* q, double* qd, double* qt, double* tips,
                          double* goals, double* axes) {
  const int T = e->T;
  for (int64_t i = 0; i < e->n; ++i) {
    for (int t = 0; t < T; ++t) {
      const int A = e->dof[t];
      for (int d = 0; d < A; ++d) {
        const int64_t k = i * e->A + e->off[t] + d;
        if (q) q[k] = e->q[t][i * A + d];
        if (qd) qd[k] = e->qd[t][i * A + d];
        if (qt) qt[k] = e->qt[t][i * A + d];
      }
      const real down[3] = {0, 0, -1};
      real ax[3];
      qrot_r(e->tquat + (i * T + t) * 4, down, ax);
      for (int k = 0; k < 3; ++k) {
        if (tips) tips[(i * T + t) * 3 + k] = e->tips[(i * T + t) * 3 + k];
        if (goals) goals[(i * T + t) * 3 + k] = e->goals[(i * T + t) * 3 + k];
        if (axes) axes[(i * T + t) * 3 + k] = ax[k];
      }
    }
  }
}

void sgo_mt_env_get_counters(const sgo_mt_env* e, int32_t* sc, int32_t* hc, int64_t* ec) {
  for (int64_t i = 0; i < e->n; ++i) {
    if (sc) sc[i] = e->step_count[i];
    if (hc) hc[i] = e->hold_count[i];
    if (ec) ec[i] = e->episode_count[i];
  }
}

void sgo_mt_env_get_rng(const sgo_mt_env* e, uint64_t* state, uint64_t* inc) {
  for (int t = 0; t < e->T; ++t)
    for (int64_t i = 0; i < e->n; ++i) {
      if (state) state[t * e->n + i] = e->rng[t][i].state;
      if (inc) inc[t * e->n + i] = e->rng[t][i].inc;
    }
}

void sgo_mt_env_workspace(const sgo_mt_env* e, double* centers, double* radius, double* bases) {
  for (int t = 0; t < e->T; ++t) {
    for (int k = 0; k < 3; ++k) {
      if (centers) centers[3 * t + k] = e->center[t][k];
      if (bases) bases[7 * t + k] = e->base[t].xyz[k];
    }
    if (bases)
      for (int k = 0; k < 4; ++k) bases[7 * t + 3 + k] = e->base[t].quat[k];
  }
  if (radius) *radius = e->radius;
}

/* ======================================================================
 * bench_sim — bench.cpp:97-135
 * ====================================================================== */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int sgo_bench_sim(const sgo_env_cfg* c, const sgo_robot* m, int64_t total_steps, int runs,
                  int threads, double* run_seconds, int64_t* run_steps) {
  for (int run = 0; run < runs; ++run) {
    sgo_env_cfg cfg = *c;
    cfg.seed = c->seed + (uint64_t)run;
    char err[256];
    sgo_env* e = sgo_env_create(&cfg, m, NULL, threads, err, sizeof(err));
    if (!e) return 2;
    sgo_pcg32 ar;
    sgo_make_stream(cfg.seed, 0xac7104, &ar);
    const int64_t count = e->n * e->A;
    double* actions = (double*)malloc((size_t)count * sizeof(double));
    int rc = sgo_env_reset(e);
    sgo_fill_uniform_actions(&ar, actions, count);
    if (!rc) rc = sgo_env_step(e, actions);
    int64_t steps = 0;
    const double t0 = now_s();
    while (!rc && steps < total_steps) {
      sgo_fill_uniform_actions(&ar, actions, count);
      rc = sgo_env_step(e, actions);
      steps += e->n;
    }
    run_seconds[run] = now_s() - t0;
    run_steps[run] = steps;
    free(actions);
    sgo_env_destroy(e);
    if (rc) return rc;
  }
  return 0;
}

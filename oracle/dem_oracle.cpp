/*
 * dem_oracle.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct fp64 CPU oracle for one DEM timestep of
 *   T. Washizawa, Y. Nakahara, "Parallel Computing of Discrete Element Method
 *   on GPU", arXiv 1301.1714  (PAPER.md in the reference mount).
 *
 * Who may use it: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load this library. The product path
 * (paper_1301_1714_b200/) never loads, links or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Build (see oracle/build.py):
 *   g++ -O2 -std=c++17 -fno-fast-math -ffp-contract=off -shared -fPIC
 * -ffp-contract=off makes every a*b+c below two rounded operations, so the
 * contact predicate and the overlap are the exact fp64 expressions DESIGN.md
 * (reading R14) defines.
 *
 * What it computes (§4.2 process flow, lines 117-131):
 *   step 2  CM[j] = cell of particle j                    (orc_hash)
 *   step 3  stable sort CM -> SCM, SCCM with Eq. 11        (orc_sort)
 *           per-cell offsets, lower_bound semantics        (orc_offsets)
 *   step 4  reorder all properties along SCCM              (inside orc_step)
 *   step 5-6 for each sorted particle, the 27 cells of Eq. 12 (orc_neighbor_cells)
 *   step 7  pair force, Eq. 1 (simple) or Eqs. 2-10 (practical)
 *   step 8  walls as particles of infinite radius
 *   step 1  update all particle properties (semi-implicit Euler; R9)
 *
 * Readings of the paper (signs, wall limits, history lifecycle ...) are the
 * ones listed in DESIGN.md "Readings" R1-R21; each is cited where used.
 *
 * Parity pins: tests/test_oracle_*.py check every function here against
 * closed forms, worked examples, invariants and brute force.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {

/* Error codes: identical numbers to the product's dem.h by design of the
 * interface (they are part of the specification, not shared code). */
enum {
  ORC_OK = 0,
  ORC_EINVAL = -1,
  ORC_EOVERFLOW = -6,
  ORC_ENONFINITE = -7,
  ORC_EESCAPED = -8,
  ORC_ECOINCIDENT = -9,
};

enum {
  ORC_MODEL_PRACTICAL = 0, /* Eqs. 2-10 */
  ORC_MODEL_SIMPLE = 1,    /* Eq. 1    */
};

enum {
  ORC_F_TRUNCATE_DT = 1u, /* reading R4: Cundall-Strack truncation when capped */
  ORC_F_CLAMP_FN = 2u,    /* reading R3 flag: no tensile F_n (Eq. 4 normal part >= 0 along -n) */
  ORC_F_BRUTE = 1u << 16, /* oracle-only: all-pairs O(N^2) detection instead of the CDG */
};

/* Wall partner ids in the history (reading R11): 0xFFFFFFF0 + w, w = 0..5 for
 * the walls -x,+x,-y,+y,-z,+z in that order. */
static const uint32_t ORC_WALL_PID0 = 0xFFFFFFF0u;

typedef struct {
  int32_t model;
  uint32_t flags;
  double dt;      /* Δt of Eq. 7 */
  double g[3];    /* gravity, once per particle (reading R2) */
  double lo[3];   /* box; the 6 walls are its faces */
  double hi[3];
  double h;       /* cell edge of the CDG (reading R15) */
  double Cn, Ct;  /* C_{k,n}, C_{k,t}  Eqs. 8-9 */
  double alpha;   /* α                 Eq. 10  */
  double mu;      /* μ                 Eq. 5   */
  double wCn, wCt, walpha, wmu; /* the same four for particle-wall pairs */
  double ksp, kda, ksh;         /* simple model, Eq. 1 */
  /* Eqs. 8-10 and 5 write C_k, α (and μ) as functions of the pair (i, j)
   * (PAPER.md:85-93): with nmat > 1 the four coefficients of a particle pair
   * are mat[(m_i * nmat + m_j) * 4 + {0: C_n, 1: C_t, 2: α, 3: μ}] for the
   * materials m_i, m_j of the two particles, and those of a particle-wall
   * pair wmat[m_i * 4 + ...] (NULL: the wall scalars above). */
  int32_t nmat;
  const double* mat;
  const double* wmat;
  /* plates (reading R23): nplates <= 10 finite two-sided rectangles, 12
   * doubles each: centre xyz, unit normal xyz, unit in-plane axis u xyz,
   * half-length along u, half-length along v = n x u, unused. History
   * partner id 0xFFFFFFF6 + k. */
  int32_t nplates;
  const double* plates;
} orc_params;

/* ---------------------------------------------------------------- grid ---- */

/* Grid dimensions n_a = floor((hi_a - lo_a)/h)  (SPEC.md:44 reading; R15). */
int orc_grid_dims(const orc_params* p, int64_t dims[3]) {
  for (int a = 0; a < 3; ++a) {
    double w = p->hi[a] - p->lo[a];
    double q = std::floor(w / p->h);
    if (!(q >= 3.0) || !(q < 2147483647.0)) return ORC_EINVAL;
    dims[a] = (int64_t)q;
  }
  return ORC_OK;
}

/* Cell triple of one position, PAPER.md:107-109 ("every particle is registered
 * to a cell that occupies its location"), with the exact fp64 definition of
 * reading R15: c_a = clamp(floor((x_a - lo_a) * (1/h)), 0, n_a - 1). */
static void cell_of(const orc_params* p, const int64_t dims[3], const double x[3],
                    int64_t c[3]) {
  double inv_h = 1.0 / p->h;
  for (int a = 0; a < 3; ++a) {
    double t = std::floor((x[a] - p->lo[a]) * inv_h);
    if (t < 0.0) t = 0.0;
    if (t > (double)(dims[a] - 1)) t = (double)(dims[a] - 1);
    c[a] = (int64_t)t;
  }
}

static int64_t linear_cell(const int64_t dims[3], const int64_t c[3]) {
  /* linearisation i + nx (j + ny k) */
  return c[0] + dims[0] * (c[1] + dims[1] * c[2]);
}

/* Step 2: CM[j] = k when the j-th particle is inside cell k. */
int orc_hash(const orc_params* p, int64_t n, const double* x, uint32_t* CM) {
  int64_t dims[3];
  if (orc_grid_dims(p, dims) != ORC_OK) return ORC_EINVAL;
  for (int64_t j = 0; j < n; ++j) {
    int64_t c[3];
    cell_of(p, dims, &x[3 * j], c);
    CM[j] = (uint32_t)linear_cell(dims, c);
  }
  return ORC_OK;
}

/* Step 3: sort CM into SCM and the map SCCM with
 * SCM[j] = CM[SCCM[j]] (Eq. 11). Ties keep the current order (reading R16):
 * std::stable_sort is the library primitive that serves as this step. */
void orc_sort(int64_t n, const uint32_t* CM, uint32_t* SCM, uint32_t* SCCM) {
  std::vector<uint32_t> idx((size_t)n);
  for (int64_t j = 0; j < n; ++j) idx[(size_t)j] = (uint32_t)j;
  std::stable_sort(idx.begin(), idx.end(),
                   [CM](uint32_t a, uint32_t b) { return CM[a] < CM[b]; });
  for (int64_t j = 0; j < n; ++j) {
    SCCM[j] = idx[(size_t)j];
    SCM[j] = CM[idx[(size_t)j]];
  }
}

/* Per-cell start offsets over SCM (reading R17):
 * off[k] = lower_bound(SCM, k) for k = 0..ncells, so cell k is
 * [off[k], off[k+1]) and off[ncells] = n. */
void orc_offsets(int64_t n, const uint32_t* SCM, int64_t ncells, uint32_t* off) {
  for (int64_t k = 0; k <= ncells; ++k) {
    const uint32_t* lb = std::lower_bound(SCM, SCM + n, (uint32_t)k);
    off[k] = (uint32_t)(lb - SCM);
  }
}

/* Eq. 12: {(l,m,n) | i-1<=l<=i+1, j-1<=m<=j+1, k-1<=n<=k+1},
 * clipped to the grid, in ascending linear cell index. Returns the count. */
int orc_neighbor_cells(const orc_params* p, int64_t cell, int64_t* out27) {
  int64_t dims[3];
  if (orc_grid_dims(p, dims) != ORC_OK) return ORC_EINVAL;
  int64_t cx = cell % dims[0];
  int64_t cy = (cell / dims[0]) % dims[1];
  int64_t cz = cell / (dims[0] * dims[1]);
  int cnt = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int64_t c[3] = {cx + dx, cy + dy, cz + dz};
        bool in = true;
        for (int a = 0; a < 3; ++a)
          if (c[a] < 0 || c[a] >= dims[a]) in = false;
        if (in) out27[cnt++] = linear_cell(dims, c);
      }
  return cnt;
}

/* ----------------------------------------------------------- predicate ---- */

/* Contact predicate of step 7's "collision detection", defined
 * in fp64 (reading R14): with Δ = x_j - x_i,
 *   d2 = (Δx*Δx + Δy*Δy) + Δz*Δz,  S = r_i + r_j,  contact <=> d2 < S*S. */
static bool in_contact(const double* xi, const double* xj, double ri, double rj,
                       double* d2_out) {
  double dx = xj[0] - xi[0], dy = xj[1] - xi[1], dz = xj[2] - xi[2];
  double d2 = (dx * dx + dy * dy) + dz * dz;
  double S = ri + rj;
  if (d2_out) *d2_out = d2;
  return d2 < S * S;
}

/* All-pairs O(N^2) detection: the plain definition of the contact set
 * ("brute-force oracle"). Writes pairs (i<j); returns count or
 * -1 if cap is too small. */
int64_t orc_contacts_brute(int64_t n, const double* x, const double* r, int64_t cap,
                           uint32_t* pi, uint32_t* pj) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j)
      if (in_contact(&x[3 * i], &x[3 * j], r[i], r[j], nullptr)) {
        if (m >= cap) return -1;
        pi[m] = (uint32_t)i;
        pj[m] = (uint32_t)j;
        ++m;
      }
  return m;
}

/* The same set through the CDG: steps 2, 3, 6. Pairs are
 * reported as original indices (i<j). */
int64_t orc_contacts_grid(const orc_params* p, int64_t n, const double* x, const double* r,
                          int64_t cap, uint32_t* pi, uint32_t* pj) {
  int64_t dims[3];
  if (orc_grid_dims(p, dims) != ORC_OK) return -2;
  int64_t ncells = dims[0] * dims[1] * dims[2];
  std::vector<uint32_t> CM((size_t)n), SCM((size_t)n), SCCM((size_t)n), off((size_t)ncells + 1);
  orc_hash(p, n, x, CM.data());
  orc_sort(n, CM.data(), SCM.data(), SCCM.data());
  orc_offsets(n, SCM.data(), ncells, off.data());
  int64_t m = 0;
  int64_t nb[27];
  for (int64_t s = 0; s < n; ++s) {
    uint32_t i = SCCM[(size_t)s];
    int k = orc_neighbor_cells(p, SCM[(size_t)s], nb);
    for (int q = 0; q < k; ++q)
      for (uint32_t t = off[(size_t)nb[q]]; t < off[(size_t)nb[q] + 1]; ++t) {
        uint32_t j = SCCM[t];
        if (j <= i) continue; /* each unordered pair once */
        if (in_contact(&x[3 * i], &x[3 * j], r[i], r[j], nullptr)) {
          if (m >= cap) return -1;
          pi[m] = i;
          pj[m] = j;
          ++m;
        }
      }
  }
  return m;
}

/* --------------------------------------------------- practical model ----- */

static inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
static inline void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
static inline double norm3(const double* a) { return std::sqrt(dot3(a, a)); }

/* Eqs. 8-9:
 *   k_t = C_{k,t} sqrt(|δ_n| / (r_i^-1 + r_j^-1)),  k_n = C_{k,n} sqrt(same).
 * Rstar = 1/(r_i^-1 + r_j^-1) is passed in so that the wall limit r_j -> ∞
 * (reading R11) can pass Rstar = r_i exactly. */
void orc_stiffness(double Cn, double Ct, double delta, double Rstar, double* kn, double* kt) {
  double s = std::sqrt(delta * Rstar);
  *kn = Cn * s;
  *kt = Ct * s;
}

/* Eq. 10: η = α sqrt(k_n / (m_i^-1 + m_j^-1)) = α sqrt(k_n m*). */
double orc_damping(double alpha, double kn, double mstar) { return alpha * std::sqrt(kn * mstar); }

/* Eq. 6: v_t = v - (v·n)n + (r_i ω_i + r_j ω_j) × n, with
 * v = v_i - v_j and n the unit vector from i to j (reading R1). */
void orc_tangential_velocity(const double* v, const double* rw, const double* n, double* vt) {
  double vn = dot3(v, n);
  double c[3];
  cross3(rw, n, c);
  for (int a = 0; a < 3; ++a) vt[a] = (v[a] - vn * n[a]) + c[a];
}

/* Eq. 7: δ_t = δ_t,old - (δ_t,old·n)n + v_t Δt. */
void orc_tangential_displacement(const double* dt_old, const double* n, const double* vt,
                                 double dt, double* dt_new) {
  double p = dot3(dt_old, n);
  for (int a = 0; a < 3; ++a) dt_new[a] = (dt_old[a] - p * n[a]) + vt[a] * dt;
}

/* Eq. 5: F_t <- μ|F_n| F_t/|F_t| if |F_t| > μ|F_n|.
 * fn_mag is |F_n| (or its clamped value under reading R3). Returns 1 if capped. */
int orc_friction_cap(double* Ft, double fn_mag, double mu) {
  double ft = norm3(Ft);
  double lim = mu * fn_mag;
  if (ft > lim) {
    double s = lim / ft;
    for (int a = 0; a < 3; ++a) Ft[a] = Ft[a] * s;
    return 1;
  }
  return 0;
}

/* One practical-model contact seen from particle i (Eqs. 2-10).
 * Inputs: n (unit, i->j), δ > 0 overlap, Rstar, mstar, v = v_i - v_j,
 * rw = r_i ω_i + r_j ω_j, r_i, the old tangential displacement, and the
 * coefficients. Outputs: F (force on i, Eq. 2), Tc = n × F_t (the torque is
 * r_i Tc, Eq. 3), and the new δ_t (Eq. 7) for the history. */
void orc_pair_practical(const double* n, double delta, double Rstar, double mstar,
                        const double* v, const double* rw, const double* dt_old,
                        double Cn, double Ct, double alpha, double mu, double dt,
                        uint32_t flags, double* F, double* Tc, double* dt_new, double* mag) {
  double kn, kt;
  orc_stiffness(Cn, Ct, delta, Rstar, &kn, &kt);          /* Eqs. 8-9 */
  double eta = orc_damping(alpha, kn, mstar);             /* Eq. 10   */
  double vt[3];
  orc_tangential_velocity(v, rw, n, vt);                  /* Eq. 6    */
  orc_tangential_displacement(dt_old, n, vt, dt, dt_new); /* Eq. 7    */
  double vnm = dot3(v, n);
  double Fn[3], Ft[3];
  for (int a = 0; a < 3; ++a) {
    /* Eq. 4 with δ_n = δ n and v_n = (v·n) n (reading R1): repulsive. */
    Fn[a] = -kn * delta * n[a] - eta * (vnm * n[a]);
    Ft[a] = -kt * dt_new[a] - eta * vt[a];
  }
  if ((flags & ORC_F_CLAMP_FN) && kn * delta + eta * vnm < 0.0) {
    /* reading R3 flag: the contact cannot pull, so a tensile
     * F_n (damping outweighing the spring while separating) is set to 0; |F_n|
     * of Eq. 5 is then 0 as well */
    for (int a = 0; a < 3; ++a) Fn[a] = 0.0;
  }
  double fn_mag = norm3(Fn);
  int capped = orc_friction_cap(Ft, fn_mag, mu); /* Eq. 5 */
  if (capped && (flags & ORC_F_TRUNCATE_DT) && kt > 0.0) {
    /* reading R4 (flag): Cundall-Strack, δ_t = -(F_t' + η v_t)/k_t */
    for (int a = 0; a < 3; ++a) dt_new[a] = -(Ft[a] + eta * vt[a]) / kt;
  }
  for (int a = 0; a < 3; ++a) F[a] = Fn[a] + Ft[a]; /* Eq. 2 */
  cross3(n, Ft, Tc);                                /* Eq. 3 without r_i */
  if (mag) {
    /* magnitudes of the terms Eq. 4 sums (the cancellation scale of a
     * floating-point evaluation of F and of F_t): |k_n δ|, |η v_n|, |k_t δ_t|, |η v_t| */
    double tt = kt * norm3(dt_new) + eta * norm3(vt);
    double nn = kn * delta + eta * std::fabs(vnm);
    mag[0] = nn + tt;
    /* F_t is bounded by μ|F_n| (Eq. 5): when capped it inherits the
     * cancellation of |F_n|, so its scale includes μ(|k_n δ| + |η v_n|) */
    mag[1] = tt + mu * nn;
  }
}

/* Eq. 1 with the SDK sign convention (reading R1):
 *   F_i = -k_sp δ n + k_da u + k_sh (u - (u·n) n),  u = v_j - v_i.
 * Gravity is applied once per particle in the integrator (reading R2). */
void orc_pair_simple(const double* n, double delta, const double* u, double ksp,
                     double kda, double ksh, double* F, double* mag) {
  double un = dot3(u, n);
  double ut[3];
  for (int a = 0; a < 3; ++a) {
    ut[a] = u[a] - un * n[a];
    F[a] = (-ksp * delta * n[a] + kda * u[a]) + ksh * ut[a];
  }
  if (mag) mag[0] = ksp * delta + kda * norm3(u) + ksh * norm3(ut); /* term magnitudes */
}

/* ---------------------------------------------------------------- step ---- */

typedef struct {
  double* x;     /* [3n] position  */
  double* v;     /* [3n] velocity  */
  double* w;     /* [3n] angular velocity ω */
  double* r;     /* [n]  radius    */
  double* m;     /* [n]  mass      */
  uint32_t* id;  /* [n]  persistent id */
  uint32_t* mat; /* [n]  material (orc_params.nmat > 1), NULL -> 0 */
} orc_state;

typedef struct {
  int32_t K;       /* capacity per particle */
  uint32_t* cnt;   /* [n] */
  uint32_t* pid;   /* [n*K] partner ids, slot-major */
  double* dt;      /* [n*K*3] δ_t,old */
} orc_hist;

typedef struct {
  uint32_t* CM;    /* [n]   step 2 (input order); may be NULL */
  uint32_t* SCCM;  /* [n]   step 3; may be NULL */
  uint32_t* off;   /* [ncells+1]; may be NULL */
  double* F;       /* [3n]  total contact force on each sorted particle (no gravity); may be NULL */
  double* T;       /* [3n]  total contact torque; may be NULL */
  double* Fabs;    /* [n]   Σ over the contacts of each particle (incl. walls) of the
                      magnitudes of the terms Eq. 4 (Eq. 1) sums: the cancellation scale
                      of the T2 tolerance's absolute floor; may be NULL */
  double* Tabs;    /* [n]   the same for r_i (n × F_t):
                      Σ r_i (|k_t δ_t| + |η v_t| + μ(|k_n δ| + |η v_n|)) */
  int64_t err[3];  /* code, sorted slot, particle id of the first error */
  int64_t n_pair_contacts;  /* ordered (i,j) particle contacts found (each pair twice) */
  int64_t n_wall_contacts;
  int64_t n_candidates;     /* j != i examined in the 27 cells */
} orc_out;

static void set_err(orc_out* o, int code, int64_t slot, uint32_t id) {
  if (o->err[0] == 0) {
    o->err[0] = code;
    o->err[1] = slot;
    o->err[2] = id;
  }
}

/* One timestep: PAPER.md §4.2 steps 2-8 then step 1, in that order (reading R9).
 * On entry the arrays hold the state in the current order; on return they hold
 * the new state in sorted (SCM) order, and hist holds the new per-slot lists.
 * `only` (may be NULL) restricts steps 5-8 and 1 to the sorted slots j with
 * only[j] != 0 — the other slots are returned reordered but not advanced
 * (used to check sampled particles of very large sets one by one). */
static int step_impl(const orc_params* p, int64_t n, orc_state* st, orc_hist* hist, orc_out* out,
                     const uint8_t* only) {
  out->err[0] = out->err[1] = out->err[2] = 0;
  out->n_pair_contacts = out->n_wall_contacts = out->n_candidates = 0;
  int64_t dims[3];
  if (orc_grid_dims(p, dims) != ORC_OK) return ORC_EINVAL;
  const int64_t ncells = dims[0] * dims[1] * dims[2];
  const int K = hist->K;
  const size_t N = (size_t)n;

  /* step 2: CM */
  std::vector<uint32_t> CM(N), SCM(N), SCCM(N), off((size_t)ncells + 1);
  orc_hash(p, n, st->x, CM.data());
  /* step 3: sort (Eq. 11) and per-cell offsets */
  orc_sort(n, CM.data(), SCM.data(), SCCM.data());
  orc_offsets(n, SCM.data(), ncells, off.data());
  if (out->CM) std::memcpy(out->CM, CM.data(), N * 4);
  if (out->SCCM) std::memcpy(out->SCCM, SCCM.data(), N * 4);
  if (out->off) std::memcpy(out->off, off.data(), ((size_t)ncells + 1) * 4);

  /* step 4: reorder all the properties along SCM */
  std::vector<double> x(3 * N), v(3 * N), w(3 * N), r(N), m(N);
  std::vector<uint32_t> id(N), mt(N, 0u), hcnt(N), hpid(N * K);
  std::vector<double> hdt(N * K * 3);
  for (size_t j = 0; j < N; ++j) {
    size_t s = SCCM[j];
    for (int a = 0; a < 3; ++a) {
      x[3 * j + a] = st->x[3 * s + a];
      v[3 * j + a] = st->v[3 * s + a];
      w[3 * j + a] = st->w[3 * s + a];
    }
    r[j] = st->r[s];
    m[j] = st->m[s];
    id[j] = st->id[s];
    if (st->mat) mt[j] = st->mat[s];
    hcnt[j] = hist->cnt[s];
    for (int k = 0; k < K; ++k) {
      hpid[j * K + k] = hist->pid[s * K + k];
      for (int a = 0; a < 3; ++a) hdt[(j * K + k) * 3 + a] = hist->dt[(s * K + k) * 3 + a];
    }
  }

  /* δ_t,old lookup by partner id (reading R10: absent -> new contact -> 0). */
  auto lookup = [&](size_t j, uint32_t pid, double* d) {
    d[0] = d[1] = d[2] = 0.0;
    for (uint32_t k = 0; k < hcnt[j]; ++k)
      if (hpid[j * K + k] == pid) {
        for (int a = 0; a < 3; ++a) d[a] = hdt[(j * K + k) * 3 + a];
        return;
      }
  };

  std::vector<double> F(3 * N, 0.0), T(3 * N, 0.0), Fabs(N, 0.0), Tabs(N, 0.0);
  std::vector<uint32_t> ncnt(N, 0), npid(N * K, 0);
  std::vector<double> ndt(N * K * 3, 0.0);
  const bool brute = (p->flags & ORC_F_BRUTE) != 0;
  const bool practical = p->model == ORC_MODEL_PRACTICAL;

  for (size_t j = 0; j < N; ++j) {
    if (only && !only[j]) continue;
    double* Fi = &F[3 * j];
    double* Ti = &T[3 * j];
    auto push_hist = [&](uint32_t pid, const double* d) -> bool {
      if ((int)ncnt[j] >= K) return false;
      npid[j * K + ncnt[j]] = pid;
      for (int a = 0; a < 3; ++a) ndt[(j * K + ncnt[j]) * 3 + a] = d[a];
      ncnt[j]++;
      return true;
    };
    /* steps 5-7: candidates of the 27 cells, ascending cell, ascending slot */
    auto visit = [&](size_t t) {
      out->n_candidates++;
      double d2;
      if (!in_contact(&x[3 * j], &x[3 * t], r[j], r[t], &d2)) return;
      if (d2 == 0.0) { /* reading R18 */
        set_err(out, ORC_ECOINCIDENT, (int64_t)j, id[j]);
        return;
      }
      out->n_pair_contacts++;
      double D = std::sqrt(d2);
      double nrm[3], delta = (r[j] + r[t]) - D;
      if (delta < 0.0) delta = 0.0;
      for (int a = 0; a < 3; ++a) nrm[a] = (x[3 * t + a] - x[3 * j + a]) / D;
      double Fc[3], mag[2] = {0.0, 0.0};
      if (practical) {
        double Rstar = 1.0 / (1.0 / r[j] + 1.0 / r[t]);
        double mstar = 1.0 / (1.0 / m[j] + 1.0 / m[t]);
        double vrel[3], rw[3], dold[3], dnew[3], Tc[3];
        for (int a = 0; a < 3; ++a) {
          vrel[a] = v[3 * j + a] - v[3 * t + a];
          rw[a] = r[j] * w[3 * j + a] + r[t] * w[3 * t + a];
        }
        lookup(j, id[t], dold);
        /* the pair's coefficients C_k(i, j), α(i, j), μ(i, j) (Eqs. 5, 8-10) */
        double Cn = p->Cn, Ct = p->Ct, alpha = p->alpha, mu = p->mu;
        if (p->nmat > 1) {
          const double* c = &p->mat[((size_t)mt[j] * (size_t)p->nmat + mt[t]) * 4];
          Cn = c[0], Ct = c[1], alpha = c[2], mu = c[3];
        }
        orc_pair_practical(nrm, delta, Rstar, mstar, vrel, rw, dold, Cn, Ct, alpha, mu, p->dt,
                           p->flags, Fc, Tc, dnew, mag);
        for (int a = 0; a < 3; ++a) Ti[a] += r[j] * Tc[a];
        Tabs[j] += r[j] * mag[1];
        if (!push_hist(id[t], dnew)) set_err(out, ORC_EOVERFLOW, (int64_t)j, id[j]);
      } else {
        double u[3];
        for (int a = 0; a < 3; ++a) u[a] = v[3 * t + a] - v[3 * j + a];
        orc_pair_simple(nrm, delta, u, p->ksp, p->kda, p->ksh, Fc, mag);
      }
      for (int a = 0; a < 3; ++a) Fi[a] += Fc[a];
      Fabs[j] += mag[0];
    };
    if (brute) {
      for (size_t t = 0; t < N; ++t)
        if (t != j) visit(t);
    } else {
      int64_t nb[27];
      int k = orc_neighbor_cells(p, SCM[j], nb);
      for (int q = 0; q < k; ++q)
        for (uint32_t t = off[(size_t)nb[q]]; t < off[(size_t)nb[q] + 1]; ++t)
          if (t != j) visit(t);
    }

    /* step 8: walls = particles of infinite radius (reading R11);
     * n points from the particle to the wall. */
    auto wall_contact = [&](const double* nrm, double delta, uint32_t pid) {
      out->n_wall_contacts++;
      double Fc[3], mag[2] = {0.0, 0.0};
      if (practical) {
        double rw[3], dold[3], dnew[3], Tc[3];
        for (int b = 0; b < 3; ++b) rw[b] = r[j] * w[3 * j + b]; /* r_w ω_w := 0 */
        lookup(j, pid, dold);
        double Cn = p->wCn, Ct = p->wCt, alpha = p->walpha, mu = p->wmu;
        if (p->nmat > 1 && p->wmat) {
          const double* c = &p->wmat[(size_t)mt[j] * 4];
          Cn = c[0], Ct = c[1], alpha = c[2], mu = c[3];
        }
        /* R* = r_i, m* = m_i, v_j = ω_j = 0: the limits r_j, m_j -> ∞ */
        orc_pair_practical(nrm, delta, r[j], m[j], &v[3 * j], rw, dold, Cn, Ct, alpha, mu, p->dt,
                           p->flags, Fc, Tc, dnew, mag);
        for (int b = 0; b < 3; ++b) Ti[b] += r[j] * Tc[b];
        Tabs[j] += r[j] * mag[1];
        if (!push_hist(pid, dnew)) set_err(out, ORC_EOVERFLOW, (int64_t)j, id[j]);
      } else {
        double u[3];
        for (int b = 0; b < 3; ++b) u[b] = -v[3 * j + b]; /* v_wall = 0 */
        orc_pair_simple(nrm, delta, u, p->ksp, p->kda, p->ksh, Fc, mag);
      }
      for (int b = 0; b < 3; ++b) Fi[b] += Fc[b];
      Fabs[j] += mag[0];
    };
    /* the 6 faces of the box, order -x, +x, -y, +y, -z, +z */
    for (int wdx = 0; wdx < 6; ++wdx) {
      int a = wdx / 2;
      bool hi_side = (wdx & 1) != 0;
      double dist = hi_side ? (p->hi[a] - x[3 * j + a]) : (x[3 * j + a] - p->lo[a]);
      if (!(r[j] > dist)) continue;
      double nrm[3] = {0.0, 0.0, 0.0};
      nrm[a] = hi_side ? 1.0 : -1.0;
      wall_contact(nrm, r[j] - dist, ORC_WALL_PID0 + (uint32_t)wdx);
    }
    /* plates (reading R23): finite two-sided rectangles, in the order given.
     * The contact point is the point of the rectangle closest to the centre;
     * contact iff its distance is below r_i. */
    for (int k = 0; k < p->nplates; ++k) {
      const double* P = &p->plates[12 * k]; /* centre, normal, u axis, half_u, half_v */
      double c[3] = {P[0], P[1], P[2]}, nn[3] = {P[3], P[4], P[5]}, uu[3] = {P[6], P[7], P[8]};
      double vv[3] = {nn[1] * uu[2] - nn[2] * uu[1], nn[2] * uu[0] - nn[0] * uu[2],
                      nn[0] * uu[1] - nn[1] * uu[0]}; /* v = n x u */
      double cp[3];  /* closest point of the rectangle */
      double du = 0.0, dv = 0.0;
      for (int b = 0; b < 3; ++b) {
        du += (x[3 * j + b] - c[b]) * uu[b];
        dv += (x[3 * j + b] - c[b]) * vv[b];
      }
      double qu = std::min(std::max(du, -P[9]), P[9]);
      double qv = std::min(std::max(dv, -P[10]), P[10]);
      double e[3], dist2 = 0.0;
      for (int b = 0; b < 3; ++b) {
        cp[b] = c[b] + qu * uu[b] + qv * vv[b];
        e[b] = cp[b] - x[3 * j + b];
        dist2 += e[b] * e[b];
      }
      double dist = std::sqrt(dist2);
      if (!(r[j] > dist)) continue;
      if (dist == 0.0) { /* centre on the plate: no direction (R18) */
        set_err(out, ORC_ECOINCIDENT, (int64_t)j, id[j]);
        continue;
      }
      double nrm[3] = {e[0] / dist, e[1] / dist, e[2] / dist};
      wall_contact(nrm, r[j] - dist, ORC_WALL_PID0 + 6u + (uint32_t)k);
    }
  }

  /* step 1 (next iteration): update all particle properties, semi-implicit
   * Euler with I = 0.4 m r^2 (reading R9). */
  for (size_t j = 0; j < N; ++j) {
    if (only && !only[j]) continue;
    double I = 0.4 * m[j] * r[j] * r[j];
    for (int a = 0; a < 3; ++a) {
      double acc = F[3 * j + a] / m[j] + p->g[a];
      v[3 * j + a] = v[3 * j + a] + acc * p->dt;
      x[3 * j + a] = x[3 * j + a] + v[3 * j + a] * p->dt;
      if (practical) w[3 * j + a] = w[3 * j + a] + (T[3 * j + a] / I) * p->dt;
    }
    for (int a = 0; a < 3; ++a) {
      if (!std::isfinite(x[3 * j + a]) || !std::isfinite(v[3 * j + a]) ||
          !std::isfinite(w[3 * j + a]))
        set_err(out, ORC_ENONFINITE, (int64_t)j, id[j]);
      else if (x[3 * j + a] < p->lo[a] - r[j] || x[3 * j + a] > p->hi[a] + r[j])
        set_err(out, ORC_EESCAPED, (int64_t)j, id[j]); /* reading R18 / SPEC.md:286 */
    }
  }

  /* write back in sorted order; history := the lists built this step (R10) */
  std::memcpy(st->x, x.data(), 3 * N * 8);
  std::memcpy(st->v, v.data(), 3 * N * 8);
  std::memcpy(st->w, w.data(), 3 * N * 8);
  std::memcpy(st->r, r.data(), N * 8);
  std::memcpy(st->m, m.data(), N * 8);
  std::memcpy(st->id, id.data(), N * 4);
  if (st->mat) std::memcpy(st->mat, mt.data(), N * 4);
  std::memcpy(hist->cnt, ncnt.data(), N * 4);
  std::memcpy(hist->pid, npid.data(), N * K * 4);
  std::memcpy(hist->dt, ndt.data(), N * K * 3 * 8);
  if (out->F) std::memcpy(out->F, F.data(), 3 * N * 8);
  if (out->T) std::memcpy(out->T, T.data(), 3 * N * 8);
  if (out->Fabs) std::memcpy(out->Fabs, Fabs.data(), N * 8);
  if (out->Tabs) std::memcpy(out->Tabs, Tabs.data(), N * 8);
  return (int)out->err[0];
}

int orc_step(const orc_params* p, int64_t n, orc_state* st, orc_hist* hist, orc_out* out) {
  return step_impl(p, n, st, hist, out, nullptr);
}

/* orc_step restricted to the sorted slots with only[j] != 0 (see step_impl). */
int orc_step_sampled(const orc_params* p, int64_t n, orc_state* st, orc_hist* hist,
                     orc_out* out, const uint8_t* only) {
  return step_impl(p, n, st, hist, out, only);
}

/* nsteps of orc_step (for long closed-form runs); stops at the first error. */
int orc_run(const orc_params* p, int64_t n, orc_state* st, orc_hist* hist, int64_t nsteps,
            orc_out* out) {
  orc_out o = *out;
  int rc = 0;
  for (int64_t s = 0; s < nsteps; ++s) {
    o.CM = nullptr;
    o.SCCM = nullptr;
    o.off = nullptr;
    o.F = (s == nsteps - 1) ? out->F : nullptr;
    o.T = (s == nsteps - 1) ? out->T : nullptr;
    o.Fabs = (s == nsteps - 1) ? out->Fabs : nullptr;
    o.Tabs = (s == nsteps - 1) ? out->Tabs : nullptr;
    rc = orc_step(p, n, st, hist, &o);
    if (rc != 0) break;
  }
  *out = o;
  return rc;
}

} /* extern "C" */

/*
 * dem.h — C ABI of the B200-native DEM timestep of
 *   T. Washizawa, Y. Nakahara, "Parallel Computing of Discrete Element Method
 *   on GPU", arXiv 1301.1714 (PAPER.md in the reference mount).
 *
 * One call of dem_step() advances the particle set by whole timesteps of the
 * paper's process flow (§4.2):
 *   step 2  correspondence map CM (cell hash)
 *   step 3  sort CM -> SCM, SCCM with SCM[j]=CM[SCCM[j]]   PAPER.md:121-123 (Eq. 11)
 *   step 4  reorder all particle properties along SCM
 *   step 5-6 thread(s) per sorted particle, 27-cell set    PAPER.md:126-127 (Eq. 12)
 *   step 7  pair contact force: Eq. 1 (simple) or Eqs. 2-10 (practical)
 *   step 8  walls as particles of infinite radius
 *   step 1  update all particle properties (integrator)
 * Readings of the paper where it is silent (signs, wall limits, integrator,
 * history lifecycle, predicate/hash precision) are DESIGN.md R1-R21.
 *
 * Conventions for every function:
 *   - returns int: DEM_OK (0) or a negative dem_error code;
 *   - SI units; parameters are fp32 as given; device state is fp32; the hash
 *     and the contact predicate are fp64 expressions of the fp32 values
 *     (R14, R15);
 *   - the handle owns every device buffer it allocates; the caller owns every
 *     array it passes in (host or device). set_* copy in (the caller may free
 *     or reuse its arrays on return); get_* copy out into caller arrays of
 *     capacity `cap` elements and return the needed count in *_out
 *     (DEM_EINVAL if too small). No caller pointer is retained across calls;
 *   - a handle is not thread-safe; all work is enqueued on the handle's
 *     stream. dem_step synchronises once at its end (unless DEM_F_ASYNC);
 *     get_* synchronise.
 */
#ifndef DEM_H
#define DEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DEM_ABI_VERSION 4u

/* Error codes. */
enum dem_error {
  DEM_OK = 0,
  DEM_EINVAL = -1,      /* bad argument: NULL, n<0, r<=0, m<=0, dt<=0, hi<=lo, grid dim < 3,
                           cell edge < 2 r_max (1+2^-10), id >= 0xFFFFFFF0 or duplicate,
                           particle centre outside the box, capacity too small */
  DEM_EABI = -2,        /* params->abi_version != DEM_ABI_VERSION */
  DEM_ENOMEM = -3,      /* device allocation failed */
  DEM_ECUDA = -4,       /* a CUDA runtime call failed (dem_last_error has the text) */
  DEM_ENCCL = -5,       /* reserved (no NCCL on the data path: the slab exchange is CUDA IPC) */
  DEM_EOVERFLOW = -6,   /* a particle had more than max_contacts contacts (history
                           capacity K). The step is rejected: the state and history stay
                           at the last completed step. */
  DEM_ENONFINITE = -7,  /* a position/velocity/angular velocity became non-finite
                           (explosion); state = last completed step */
  DEM_EESCAPED = -8,    /* a centre moved beyond a wall by more than its radius
                           (tunnelling); state = last completed step */
  DEM_ECOINCIDENT = -9, /* two centres coincide while in contact (n undefined, R18) */
  DEM_ESTATE = -10,     /* call out of order (e.g. dem_step before dem_set_particles) */
  DEM_EPEER = -11,      /* slab exchange failed: a neighbour did not publish in time, or a
                           particle moved more than one cell plane across a slab boundary */
};

enum dem_model {
  DEM_MODEL_PRACTICAL = 0, /* Eqs. 2-10: Hertzian spring-dashpot, Coulomb
                              cap, tangential history, torque and angular velocity */
  DEM_MODEL_SIMPLE = 1,    /* Eq. 1: linear spring, damping, shear */
};

enum dem_flags {
  DEM_F_TRUNCATE_DT = 1u << 0, /* R4: δ_t = -(F_t' + η v_t)/k_t when Eq. 5 caps F_t */
  DEM_F_CLAMP_FN = 1u << 1,    /* R3 flag: no tensile F_n (Eq. 4), so |F_n| >= 0 in Eq. 5 */
  DEM_F_DIAG = 1u << 2,        /* keep per-particle F and T of the last step (dem_get_state) */
  DEM_F_ASYNC = 1u << 3,       /* dem_step does not synchronise; errors surface at the next
                                  synchronising call */
  DEM_F_NO_GRAPH = 1u << 4,    /* launch kernels eagerly instead of replaying a CUDA graph */
  DEM_F_THREAD_PER_PARTICLE = 1u << 5, /* ablation: the paper's mapping, detection and forces
                                          in one thread-per-particle kernel */
  DEM_F_HALF_LISTS = 1u << 6, /* ablation: each contact pair evaluated once (Newton's third
                                 law, half contact lists + a per-pair result buffer); default:
                                 full lists, each side evaluated by its particle's warp */
  DEM_F_FORCE_DENSE = 1u << 7, /* force-kernel configuration for many contacts per particle;
                                  default: chosen after the first step from the measured
                                  history entries per particle (> 7: dense). Both give
                                  bitwise-identical results */
  DEM_F_FORCE_LIGHT = 1u << 8, /* force-kernel configuration for few contacts per particle */
  DEM_F_GENERAL_DETECT = 1u << 9, /* ablation: the candidate test evaluates S = r_i + r_j per
                                     pair even when every radius is equal; default (single
                                     GPU, one radius): S² is one constant. Same contact lists */
  DEM_F_FULL_SORT = 1u << 10, /* ablation: the counting sort every step; default (single GPU):
                                 a merge of the particles that changed cell into the last
                                 sorted order. Bit-identical SCCM and offsets */
  DEM_F_FORCE_LANES = 1u << 11, /* force-kernel configuration: one thread per particle over its
                                   contact list (bitwise-identical results) */
  DEM_F_FORCE_WS = 1u << 12,    /* ablation: warp-specialised force kernel (producer warps load,
                                   consumer warps compute; bitwise-identical results) */
  DEM_F_SPLIT_SWEEP = 1u << 13, /* detection (steps 5-6) as its own kernel writing contact lists
                                   to HBM; default with one radius: each force warp detects its
                                   own contacts into shared memory first (one fused kernel).
                                   Same contact lists and bitwise-identical results */
};

enum dem_mem_kind { DEM_MEM_HOST = 0, DEM_MEM_DEVICE = 1 };
enum dem_order {
  DEM_ORDER_INTERNAL = 0, /* the handle's current memory order = SCM order of the last sort */
  DEM_ORDER_ID = 1,       /* by persistent id; requires ids to be a permutation of 0..n-1 */
};

typedef struct dem_handle dem_handle; /* opaque; owns all device memory */

/* Optional device-memory provider (torch passes its caching allocator). */
typedef struct {
  void* ctx;
  void* (*alloc)(void* ctx, size_t bytes, void* stream);
  void (*free)(void* ctx, void* ptr, size_t bytes, void* stream);
} dem_allocator;

/* The paper's problem statement: radius, spring
 * parameters C_k, restitution parameter α, friction μ, gravity, Δt, walls,
 * and the simple model's constants. */
typedef struct {
  uint32_t abi_version;      /* == DEM_ABI_VERSION, else DEM_EABI */
  int32_t model;             /* enum dem_model */
  float dt;                  /* Δt > 0 [s] (Eq. 7) */
  float gravity[3];          /* g [m/s^2], applied once per particle (R2) */
  float box_lo[3];           /* domain; the 6 walls are its faces */
  float box_hi[3];
  float radius;              /* default radius when dem_particles.radius == NULL [m] */
  float density;             /* default mass = density (4/3) π r^3 when mass == NULL */
  float stiffness_n;         /* C_{k,n} [Pa]  (Eq. 9)  */
  float stiffness_t;         /* C_{k,t} [Pa]  (Eq. 8)  */
  float damping;             /* α             (Eq. 10) */
  float friction;            /* μ             (Eq. 5)  */
  float wall_stiffness_n;    /* the same for particle-wall pairs; < 0 -> particle value */
  float wall_stiffness_t;
  float wall_damping;
  float wall_friction;
  float k_sp, k_da, k_sh;    /* simple model (Eq. 1) [N/m, N s/m, N s/m] */
  float cell_edge;           /* CDG cell edge h; 0 -> 2 r_max (1 + 2^-10) in fp64 (R15) */
  uint32_t max_contacts;     /* history capacity K per particle; 0 -> 16; <= 64 (else DEM_EINVAL;
                                <= 32 with DEM_F_HALF_LISTS) */
  uint32_t flags;            /* enum dem_flags */
  int32_t device;            /* CUDA ordinal; -1 -> current device */
  void* stream;              /* cudaStream_t; NULL -> a stream owned by the handle */
  const dem_allocator* allocator; /* NULL -> cudaMallocAsync on the stream */
  int32_t rank, world_size;  /* world_size <= 1: single GPU; > 1: z-slab rank */
  /* Eqs. 5, 8-10 write C_k, α (and μ) as functions of the pair (i, j)
   * (PAPER.md:85-93). n_materials <= 1: the scalars above for every pair.
   * 2 <= n_materials <= 16: material_pairs (host, [M][M][4] = C_n, C_t, α, μ,
   * symmetric, finite, >= 0) gives each particle pair its coefficients from
   * the two particles' materials (dem_particles.material); material_walls
   * (host, [M][4], or NULL for the wall scalars above) those of a
   * particle-wall pair. Ids must then be < 2^27 (the material travels in the
   * id word's bits 27-30). Copied at dem_create. */
  uint32_t n_materials;
  const float* material_pairs;
  const float* material_walls;
  /* Walls besides the box faces (reading R23, e.g. the §5 box with a slit,
   * PAPER.md:139): n_plates <= 10 finite two-sided rectangles, plates = host
   * [n_plates][12]: centre xyz, unit normal xyz, unit in-plane axis u xyz,
   * half-length along u, half-length along v = normal x u, unused. A plate
   * is a particle of infinite radius (R11) touching at the rectangle's point
   * closest to the centre; wall coefficients; history partner id
   * 0xFFFFFFF6 + k. Copied at dem_create. */
  uint32_t n_plates;
  const float* plates;
} dem_params;

/* Particle arrays, all host or all device (mem_kind). Layout: pos/vel/omega
 * are [3n] xyz-interleaved float; radius/mass [n]; id [n]. For
 * dem_set_particles a NULL member means "default" (vel, omega = 0; radius =
 * params.radius; mass from density; id = 0..n-1). For dem_get_state a NULL
 * member is not written. force/torque are output-only (DEM_F_DIAG): the
 * contact force and torque of the last evaluated step, without gravity. */
typedef struct {
  int32_t mem_kind;
  float* pos;
  float* vel;
  float* omega;
  float* radius;
  float* mass;
  uint32_t* id;
  float* force;
  float* torque;
  uint32_t* material;        /* [n] material ids < n_materials; NULL -> 0 (in) / not written (out) */
} dem_particles;

typedef struct {
  int64_t n;             /* particles held by this handle */
  int64_t ncells;        /* CDG cells */
  int32_t dims[3];       /* CDG dimensions */
  double cell_edge;      /* h actually used */
  int64_t steps;         /* completed steps since dem_set_particles */
  int64_t contacts;      /* history entries (= 2 pair contacts + wall contacts) of the last step */
  int64_t max_contacts_seen; /* max per-particle history entries of the last step */
  int64_t launches;      /* kernels this handle launched since creation */
  int64_t graph_launches;
  /* per-kernel device time accumulated while profiling (dem_profile) */
  double kernel_ms[8];
  int64_t kernel_count[8];
  int32_t force_cfg;     /* force configuration in use: 0 dense, 1 light, 2 lanes, -1 not chosen yet */
  int32_t full_sorts;    /* steps sorted by the counting sort since dem_set_particles: the
                            first, and any in which more than max(4,096, n/512) particles
                            changed cell (slab ranks: plus twice the migrant capacity);
                            the others merge the few movers into the last sorted order */
  double max_speed;      /* max |v| of the current state [m/s]: the last step moved no
                            particle farther than max_speed * dt (the §5 termination test) */
  int32_t fused_sweep;   /* 1: detection (steps 5-6) runs inside the force kernel (one radius,
                            no DEM_F_SPLIT_SWEEP or ablation flag); 0: k_detect + k_force */
  int32_t reserved;
} dem_stats;

/* Kernel indices of dem_stats.kernel_ms. Counting sort: DEM_K_HASH cell
 * counts (k_count, merge mode's counting steps only), DEM_K_SCAN offsets,
 * DEM_K_SCATTER, DEM_K_RANK; merge re-sort: DEM_K_SCATTER the movers' sort
 * (k_mv_sort), DEM_K_RANK the merge and offset shifts (k_mv_apply). */
enum dem_kernel { DEM_K_HASH = 0, DEM_K_SCAN = 1, DEM_K_SCATTER = 2, DEM_K_RANK = 3,
                  DEM_K_SWEEP = 4 /* contact forces (k_pair, or the fused sweep) */,
                  DEM_K_OTHER = 5 /* slab exchange, introspection */,
                  DEM_K_DETECT = 6 /* contact detection */,
                  DEM_K_FINISH = 7 /* per-particle sums, walls, integration */ };

/* Create a handle: validates params (DEM_EINVAL/DEM_EABI), selects the device
 * and stream. Grid and buffers are sized by dem_set_particles. *out = NULL on
 * error. */
int dem_create(const dem_params* p, dem_handle** out);

/* Release every device buffer and the owned stream. NULL is a no-op. */
int dem_destroy(dem_handle* h);

/* Copy in n particles ("particle properties") and clear the
 * contact history. Validates radius > 0, mass > 0, finite values, centres
 * at most r beyond a wall (R18: what a step may produce), ids < 0xFFFFFFF0
 * and unique, and the cell edge against
 * 2 r_max (1 + 2^-10). Sizes the CDG: n_a = floor((hi_a - lo_a)/h) >= 3.
 * Computes CM for the next step (step 2). n == 0 is allowed. */
int dem_set_particles(dem_handle* h, int64_t n, const dem_particles* src);

/* Replace the tangential-displacement history (Eq. 7's δ_t,old) with m
 * entries (id_i, id_j, dt3[3]): the displacement stored on particle id_i's
 * side for partner id_j (a wall w = 0..5 is id 0xFFFFFFF0 + w). Arrays are
 * host or device per mem_kind. Single GPU: requires dense ids (a permutation
 * of 0..n-1; an id_i outside is DEM_EINVAL). Slab rank (world_size > 1): ids
 * below 4 n + 2^20 of the set passed to dem_set_particles; entries whose
 * id_i this rank does not own are skipped, so every rank may be given the
 * same global list (or only its own, e.g. its dem_get_contacts output).
 * DEM_EOVERFLOW if a particle gets more than max_contacts entries. */
int dem_set_contacts(dem_handle* h, int32_t mem_kind, int64_t m, const uint32_t* id_i,
                     const uint32_t* id_j, const float* dt3);

/* Advance nsteps >= 0 timesteps. On an error code the state and history are
 * those of the last completed step and dem_last_error() names the particle
 * and step. */
int dem_step(dem_handle* h, int64_t nsteps);

/* Wait for enqueued work; returns a pending step error (DEM_F_ASYNC). */
int dem_sync(dem_handle* h);

/* Copy out the state (order: enum dem_order). *n_out = n. */
int dem_get_state(dem_handle* h, int32_t order, int64_t cap, const dem_particles* dst,
                  int64_t* n_out);

/* Copy out the history as (id_i, id_j, dt3) triples, grouped by particle in
 * internal order, each particle's entries in the order the step found them
 * (27 cells ascending, slots ascending, then walls -x,+x,-y,+y,-z,+z).
 * mem_kind says where the output arrays live. *m_out = number of entries. */
int dem_get_contacts(dem_handle* h, int32_t mem_kind, int64_t cap, uint32_t* id_i,
                     uint32_t* id_j, float* dt3, int64_t* m_out);

/* Diagnostics for bit-exact checks (host arrays; any may be NULL):
 *   key [n]        CM of the current state (what the next step will sort)
 *   perm [n]       SCCM of the last sort (Eq. 11), i.e. the old slot of each new slot
 *   off [ncells+1] cell start offsets of the last sort (lower_bound semantics)
 * cap bounds perm/key (n) and off (ncells+1). *ncells_out = ncells. */
int dem_get_grid(dem_handle* h, int64_t cap, uint32_t* key, uint32_t* perm, uint32_t* off,
                 int64_t* ncells_out);

/* Counters (see dem_stats). Synchronises; computes the contact totals from
 * the current history with a small reduction kernel. */
int dem_get_stats(dem_handle* h, dem_stats* out);

/* The quantities of the paper's §6 analysis, measured on
 * the input state of the last step (its sort, cell offsets and contact
 * lists; owned slots only in slab mode). "Warp" = 32 consecutive sorted
 * slots, the thread-per-particle mapping of the paper (and of k_detect). */
typedef struct {
  int64_t n;                 /* particles analysed */
  int64_t candidates;        /* Σ_i particles j != i in i's 27 cells (Eq. 12; "about 47") */
  int64_t max_candidates;
  int64_t contacts;          /* Σ_i particle-particle contacts of i (walls excluded) */
  int64_t max_contacts;      /* the kissing bound is 12 for equal spheres */
  int64_t warp_candidate_slots; /* Σ_warps 32 · max_lanes candidates: lane-iterations of the
                                   candidate loop under SIMT (divergence) */
  int64_t warp_contact_slots;   /* Σ_warps 32 · max_lanes contacts: lane-iterations of the
                                   contact-force evaluation if done per thread */
  int64_t max_per_cell;      /* most particles in one cell (Eq. 13: √2 (h/d)³ at close packing) */
  int64_t occupied_cells;
  int64_t contact_hist[33];  /* particles with k contacts, k = 0..31; [32]: 32 or more */
  int64_t movers;            /* particles the last step moved to another cell (the next merge
                                re-sort's input); -1 without the merge re-sort (slabs,
                                DEM_F_FULL_SORT) */
} dem_analysis;

/* Fill *out from the last step (DEM_ESTATE before the first step).
 * Synchronises; one small kernel. */
int dem_analyze(dem_handle* h, dem_analysis* out);

/* Per-kernel CUDA-event timing of subsequent dem_step calls (eager launches,
 * events around every kernel on the handle's stream); 0 disables. Enabling
 * resets the accumulated times. */
int dem_profile(dem_handle* h, int32_t enable);

/* ---- Slab decomposition (world_size > 1) ---------------------
 * Rank r of P owns the cell planes z in [floor(r nz/P), floor((r+1) nz/P)) of
 * the global grid (nz >= 2P). dem_set_particles takes the full set (or any
 * superset of the rank's slab) and keeps the rank's particles. Every step
 * starts by reading the neighbours' migrants and ghost planes from their
 * exchange regions (peer memory over NVLink via CUDA IPC) and ends by
 * publishing this rank's. Ranks must be connected before dem_step, and step
 * in lockstep (a rank waits for its neighbours' previous step). After a step,
 * dem_get_state / dem_get_contacts return the particles this rank advanced;
 * the union over ranks is the whole set, each particle exactly once. Errors
 * in slab mode are not rolled back (set the particles again). */

/* 64-byte cudaIpcMemHandle_t of this rank's exchange region (after
 * dem_set_particles); the caller distributes it to the neighbours. */
int dem_exchange_handle(dem_handle* h, void* out64);
/* Device pointer of the exchange region (same-process neighbours). */
int dem_exchange_ptr(dem_handle* h, void** out);
/* Open the neighbours' handles (NULL for rank 0's left / rank P-1's right). */
int dem_connect(dem_handle* h, const void* left64, const void* right64);
/* Same-process neighbours: their dem_exchange_ptr values (NULL at the ends). */
int dem_connect_ptrs(dem_handle* h, void* left, void* right);

const char* dem_strerror(int code);
/* Text of the last error on this handle (includes particle id and step for
 * DEM_ENONFINITE / DEM_EESCAPED / DEM_EOVERFLOW / DEM_ECOINCIDENT). */
const char* dem_last_error(const dem_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* DEM_H */

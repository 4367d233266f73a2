// dem_internal.h — device-side data layout and kernel launchers of libdem.so.
// Product code (the CUDA path). Shares nothing with oracle/.
//
// HBM layout, per particle slot j of buffer b in {0,1}:
//   pos_r[b][j]  = (x, y, z, r)                      float4
//   vel_m[b][j]  = (vx, vy, vz, m)                   float4
//   omg_id[b][j] = (wx, wy, wz, bits(id))            float4
//   key[b][j]    = CM (cell of this slot's position) u32
//   hist[b][j*K + k] = (δt_x, δt_y, δt_z, bits(pid)) float4, k < cnt[b][j] <= K (slot-major)
// and, per step: prank[N] (rank of a slot inside its cell from the counting
// atomics), count[ncells] (particles per cell, zero between steps),
// off[ncells+1] (= exclusive scan of count = lower_bound offsets of SCM),
// tmp[N] (slots scattered by cell, unordered inside a cell) and perm[N]
// (= SCCM of Eq. 11: old slot of each new slot, stable).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dem {

constexpr uint32_t kWallPid0 = 0xFFFFFFF0u;
constexpr uint32_t kMaxContacts = 64;  // largest list capacity K dem_create accepts

struct DevGrid {
  int nx, ny, nz;    // local grid (nz = planes held by this rank, ghosts included)
  uint32_t ncells;   // local cells (+1 trash cell for departed particles in slab mode)
  double lo[3], hi[3];
  double inv_h;      // 1/h, correctly rounded on the host (R15)
  int nz_global;     // global planes along z
  int zlo;           // global z of local plane 0
  int z0, z1;        // global z range [z0, z1) owned by this rank (single GPU: [0, nz))
  uint32_t own_c0, own_c1;  // local cells of the owned planes: owned sorted slots are
                            // [off[own_c0], off[own_c1])
  uint32_t trash;    // key of particles outside the local grid (slab mode), else ncells
  int slab;          // 1: slab decomposition active
  uint32_t xbase;    // slab exchange tags = xbase + step number (distinct across re-sets)
};

struct DevPhys {
  float dt;
  float g[3];
  float Cn, Ct, alpha, mu;
  float wCn, wCt, walpha, wmu;
  float ksp, kda, ksh;
  uint32_t flags;
  // material pairs (dem_params.n_materials > 1): coefficients (C_n, C_t, α, μ)
  // of a particle pair mat[m_i * nmat + m_j], of a particle-wall pair wmat[m_i];
  // the material is bits 27-30 of the id word (omg.w), idmask strips it
  const float4* mat;
  const float4* wmat;
  uint32_t nmat;
  uint32_t idmask;  // 0x07FFFFFF with materials, else 0xFFFFFFFF
  // plates (R23): nplates finite two-sided rectangles, 12 floats each
  const float* plates;
  uint32_t nplates;
};
constexpr uint32_t kMatShift = 27;

// Device error record. code is the positive value of the dem_error.
struct DevErr {
  uint32_t code;
  uint32_t slot;
  uint32_t id;
  uint32_t step;      // value of step_ctr in the failing step
  uint32_t step_ctr;  // steps started since dem_set_particles (incremented by k_scan)
  uint32_t pad[3];
};

// Status words of the decoupled look-back scan: [flag:2 | value:32].
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

// merge re-sort (k_merge): mover lists double-buffered by the
// parity of the state they index
struct MergeBuffers {
  const uint4* list_in;   // movers of this step's input order, listed by the previous
                          // step's integrator: (slot, new key, previous key, insertion point)
  const uint32_t* n_in;   // their number (may exceed cap: the step is redone by counting)
  uint4* list_out;        // this step's integrator lists the next step's movers here
  uint32_t* n_out;        // (zeroed by this step's k_merge, or memset on a counting step)
  uint32_t cap;           // list capacity
};

struct StepBuffers {
  const float4* pos_in;
  const float4* vel_in;
  const float4* omg_in;
  float4* pos_out;
  float4* vel_out;
  float4* omg_out;
  const uint32_t* key_in;
  uint32_t* key_out;
  uint32_t* prank;
  uint32_t* count;
  uint32_t* off;
  uint32_t* tmp;
  uint32_t* perm;
  float4* pos_sorted;  // (x,y,z,r) gathered into SCM order by k_rank (step 4, positions)
  float sw_r;          // > 0: one radius sw_r and the default path: pos_sorted[j].w holds
                       // bits(SCCM[j]) instead of r (the contact lists then carry old slots)
  uint32_t* clist;     // contacts found by k_detect: clist[k*N + j] = partner's sorted slot
  uint32_t* ccount;    // per owned slot, from k_detect: base | n << 16 | overflow << 31 (its
                       // first contact in its warp's flattened order, its contacts n <= K,
                       // more than K found); the half-list ablation keeps a plain count
  const uint32_t* nslots;  // device: input slots of this step (owned + appended)
  uint32_t* flags;     // slab mode: per output slot, bit0/1 migrate to left/right neighbour,
                       // bit2/3 ghost for left/right neighbour
  uint32_t* xtc;       // slab mode: [4][xntiles] flagged outputs per category and pack tile
                       // (kXTile output slots), [xntiles] flagged outputs per tile, then the
                       // number of tiles with any: accumulated by this step's integrator,
                       // read by its pack (one buffer per state parity)
  uint32_t* xtc_next;  // the other parity's: zeroed by this step's pack for the next step
  uint32_t xntiles;
  uint32_t gl_base;    // first sorted slot of the owned particles: a slab rank with a left
                       // neighbour keeps room below it for the left ghost plane (placed
                       // right-aligned); else 0
  // half-list path (Newton's third law): the pair (i, t) is
  // evaluated once, by its lower sorted slot i ("upper" contact of i)
  uint8_t* cpos;       // [k*N + i]: position of i in t's lower list
  uint32_t* lcount;    // [t]: lower contacts appended to t (atomics in k_detect_half)
  uint32_t* llist;     // [p*N + t] = i << 5 | k: t's lower contact p is i's upper contact k
  float4* R0;          // [k*N + i]: (F_c on i, Tc.x) of i's upper contact k
  float2* R1;          // [k*N + i]: (Tc.y, Tc.z)
  const float4* hist_in;
  const uint32_t* cnt_in;
  float4* hist_out;
  uint32_t* cnt_out;
  float4* F_out;  // DEM_F_DIAG only
  float4* T_out;
  unsigned long long* scan_status;       // the counting sort's tile sums (this parity's)
  DevErr* err;
  // merge re-sort (single GPU): the mover buffers
  // (mv.mov == nullptr: counting sort, cell counts)
  MergeBuffers mv;
};
// movers per step the merge re-sort takes: a few per mille of the particles
// move cell per step on the settling bed (C4: ~500 of 4.2 M)
inline uint32_t mover_cap(int64_t n) {
  const int64_t c = n / 512;
  return (uint32_t)(c < 4096 ? 4096 : c > 65536 ? 65536 : c);
}

// ---- slab exchange ------------------------------------------
// Per rank an exchange region (cudaMalloc, shareable by CUDA IPC) holding, for
// each direction d (0 = to the left neighbour, 1 = to the right) and step
// parity p, a header and the packed migrants (state + history) and ghosts
// (state) of that step. The neighbour reads it directly (peer memory).
struct XHeader {
  uint32_t tag;     // step number the data is for (published last, release/acquire)
  uint32_t n_mig;   // migrants packed
  uint32_t n_ghost; // the sender's boundary plane for the next step, sorted by its keys
  uint32_t pad;
};
constexpr uint32_t kXTile = 1024;  // output slots per pack tile (256 threads x 4)
// per state parity: tile counts [4][ntiles], per-tile sums [ntiles], the
// number of tiles with flagged outputs (+ padding)
inline uint32_t xtc_ntiles(int64_t cap) { return (uint32_t)((cap + kXTile - 1) / kXTile); }
inline uint32_t xtc_stride(int64_t cap) { return 5u * xtc_ntiles(cap) + 4u; }
// An exchange region = a header holding the writer's XLayout (read by the
// neighbours at connect time) + 4 blocks (direction x parity).
constexpr uint64_t kXRegionHdr = 256;
constexpr uint32_t kXPoison = 0xFFFFFFFFu;  // XHeader.n_mig of a failed step's publication
struct XLayout {  // byte offsets inside one (direction, parity) block
  uint64_t header, mig_pos, mig_vel, mig_omg, mig_cnt, mig_hist, gh_pos, gh_vel, gh_omg, gh_off,
      bytes;
  uint32_t mig_cap, ghost_cap, K;
  uint32_t plane;      // cells per z-plane: the ghost plane's cell offsets hold plane + 1
  uint32_t mono_bits;  // the set's one radius (bits; 0: several): neighbours must agree
  __host__ __device__ static XLayout make(uint32_t mig_cap, uint32_t ghost_cap, uint32_t K,
                                          uint32_t plane) {
    XLayout L;
    L.mig_cap = mig_cap;
    L.ghost_cap = ghost_cap;
    L.K = K;
    L.plane = plane;
    L.mono_bits = 0;
    uint64_t o = 0;
    L.header = o;
    o += 256;
    L.mig_pos = o;
    o += (uint64_t)mig_cap * 16;
    L.mig_vel = o;
    o += (uint64_t)mig_cap * 16;
    L.mig_omg = o;
    o += (uint64_t)mig_cap * 16;
    L.mig_cnt = o;
    o += ((uint64_t)mig_cap * 4 + 255) & ~255ull;
    L.mig_hist = o;  // entry-major: [m * K + k]
    o += (uint64_t)mig_cap * K * 16;
    L.gh_pos = o;
    o += (uint64_t)ghost_cap * 16;
    L.gh_vel = o;
    o += (uint64_t)ghost_cap * 16;
    L.gh_omg = o;
    o += (uint64_t)ghost_cap * 16;
    L.gh_off = o;  // the plane's cell offsets, relative to its first particle
    o += ((uint64_t)(plane + 1) * 4 + 255) & ~255ull;
    L.bytes = (o + 4095) & ~4095ull;
    return L;
  }
};
struct XState {  // device scratch of the exchange of one step
  uint32_t n_out;      // output slots of the last step (base of the appended slots)
  uint32_t appended[4];  // migrants from left, right; ghosts from left, right
  uint32_t done;       // pack blocks finished this step (the last one publishes)
  uint32_t pad[2];     // pad[0]: this step's exchange tag (set by k_xrecv)
};

enum KernelId { K_HASH = 0, K_SCAN = 1, K_SCATTER = 2, K_RANK = 3, K_SWEEP = 4, K_OTHER = 5,
                K_DETECT = 6, K_FINISH = 7 };

// ---- launchers (dem_kernels.cu) -------------------------------------------
// Every launcher enqueues exactly one kernel on `st` and returns its id.

// set_particles: AoS inputs (device) -> SoA float4 slots, CM, counting ranks.
struct PackIn {
  const float* pos;
  const float* vel;
  const float* omega;
  const float* radius;
  const float* mass;
  const uint32_t* id;
  const uint32_t* material;  // NULL -> 0
  float def_radius, def_mass_coef;  // mass = coef * r^3 when mass == NULL
  uint32_t nmat;                    // > 1: material stored in the id word's bits 27-30
};
struct Probe {  // validation results of k_probe
  uint32_t bad_radius, bad_mass, nonfinite, outside, bad_id;
  uint32_t rmax_bits, id_max, bad_material;
  uint32_t rmin_cbits;  // max of ~bits(r): r_min = ~rmin_cbits (zero-initialised like the rest)
};
int launch_probe(cudaStream_t st, int64_t n, PackIn in, DevGrid g, Probe* out);
int launch_pack(cudaStream_t st, int64_t n, PackIn in, DevGrid g, float4* pos, float4* vel,
                float4* omg, uint32_t* key, uint32_t* count, uint32_t* prank,
                const uint32_t* dst = nullptr, const uint32_t* keep = nullptr);
// initial exchange flags of the set state (slab mode)
int launch_flags(cudaStream_t st, int64_t n, const float4* pos, DevGrid g, uint32_t* flags);
int launch_count(cudaStream_t st, int64_t n, const uint32_t* key, uint32_t* count,
                 uint32_t* prank);
int launch_idcheck(cudaStream_t st, int64_t n, uint32_t idmask, const float4* omg, uint32_t* seen,
                   uint32_t* dup_flag);

// One step = scan, scatter, rank, sweep.
int launch_scan(cudaStream_t st, const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* zero,
                unsigned long long* status, uint32_t* ctr, DevErr* err, int count_step,
                uint32_t base0 = 0);  // base0: added to every output (the owned particles' start)
int launch_scatter(cudaStream_t st, int64_t n, const StepBuffers& b);
int launch_rank(cudaStream_t st, int64_t n, const StepBuffers& b);
// merge re-sort: one k_merge in place of the counting sort
// when the state is in the previous step's sorted order
// Slab ranks (g.slab): the owned particles — n read from n_dev (the last
// step's outputs; the host n is the grid's bound), placed from b.gl_base,
// offsets of the owned cells only; list entries with insertion point
// 0xFFFFFFFF (migrants that left) are removals, entries with previous key
// 0xFFFFFFFF (migrants that arrived) insertions
// L non-null (slab): the ghost planes are placed by extra blocks of the same
// kernel (k_xghost_place's work, the owned end counted from the mover list)
int launch_merge(cudaStream_t st, int64_t n, uint32_t ncells, const StepBuffers& b,
                 const DevGrid& g, const uint32_t* n_dev = nullptr,
                 const uint8_t* left = nullptr, const uint8_t* right = nullptr,
                 const XLayout* L = nullptr, XState* xs = nullptr);
int launch_perm_from_w(cudaStream_t st, int64_t n, const float4* pos_sorted, uint32_t* perm);
// Default: k_detect (steps 5-6: contact lists) then k_force (steps 7-8 + 1,
// warp-cooperative). Variant 1 (ablation): one thread per particle for the
// whole step (the paper's mapping) in a single kernel.
void sweep_prepare(uint32_t K);  // host: kernel attributes (call outside stream capture)
// whether this library carries the ablation kernels (DEM_F_THREAD_PER_PARTICLE,
// DEM_F_HALF_LISTS, DEM_F_FORCE_LANES): libdem_ablations.so yes, libdem.so no
bool ablations_built();
// mono_r > 0: every particle has radius mono_r (single GPU), so S² of R14 is one
// constant and the fp32 candidate test is 3 instructions shorter (same decisions).
int launch_detect(cudaStream_t st, int64_t n, uint32_t K, const StepBuffers& b,
                  const DevGrid& g, float mono_r = 0.f, bool light = false);
// half-list path (default): k_detect_half, k_pair, k_finish
int launch_detect_half(cudaStream_t st, int64_t n, uint32_t K, const StepBuffers& b,
                       const DevGrid& g);
int launch_pair(cudaStream_t st, int64_t n, uint32_t K, int model, const StepBuffers& b,
                const DevGrid& g, const DevPhys& ph);
int launch_finish(cudaStream_t st, int64_t n, uint32_t K, int model, bool diag,
                  const StepBuffers& b, const DevGrid& g, const DevPhys& ph);
int launch_sweep(cudaStream_t st, int64_t n, uint32_t K, int model, bool diag,
                 const StepBuffers& b, const DevGrid& g, const DevPhys& ph, int variant);

// Slab exchange. `mine` = this rank's exchange region; `left`/`right` = the
// neighbours' regions (peer pointers, NULL at the ends of the domain).
// step end: the two boundary planes as they will be sorted next step (a
// merge of the plane's stayers with its movers, from the mover list) and
// the migrants; the last block releases the tag. initial = 1: the set state
// (sorted already at set time: its sorted runs are published as they are)
int launch_xpack(cudaStream_t st, int64_t cap, const StepBuffers& b, const DevGrid& g, uint32_t K,
                 uint8_t* mine, XLayout L, XState* xs, int initial, int nbr);
// step start: acquire the neighbours' tags; append their migrants (state +
// history) at slots n_out.. (merge step: listed as insertions; counting
// step: counted into their cells) and their boundary planes' state after them
int launch_xrecv(cudaStream_t st, int64_t cap, const StepBuffers& b, const DevGrid& g, uint32_t K,
                 const uint8_t* left, const uint8_t* right, XLayout L, XState* xs,
                 uint32_t* nslots_out, bool merge);
// after the owned sort: the received planes as this rank's ghost planes,
// merged with its own departed particles (sorted slots right-aligned below
// gl_base and right after the owned particles), and the ghost cells' offsets
int launch_xghost_place(cudaStream_t st, int64_t cap, const StepBuffers& b, const DevGrid& g,
                        const uint8_t* left, const uint8_t* right, XLayout L, XState* xs);
// set_particles in slab mode: keep[i] = particle i's z-cell is owned by this rank.
int launch_keep(cudaStream_t st, int64_t n, const float* pos, DevGrid g, uint32_t* keep);
int launch_plane_hist(cudaStream_t st, int64_t n, const float* pos, DevGrid g, uint32_t* hist);

// Introspection / state movement.
int launch_unpack(cudaStream_t st, int64_t n, bool by_id, const float4* pos, const float4* vel,
                  const float4* omg, const float4* F, const float4* T, float* o_pos,
                  float* o_vel, float* o_omg, float* o_r, float* o_m, uint32_t* o_id,
                  float* o_F, float* o_T, uint32_t idmask, uint32_t* o_mat);
int launch_emit_contacts(cudaStream_t st, int64_t n, int64_t stride, uint32_t K,
                         const float4* hist, const uint32_t* cnt, const uint32_t* base,
                         const float4* omg, uint32_t* id_i, uint32_t* id_j, float* dt3,
                         uint32_t idmask);
int launch_slot_of_id(cudaStream_t st, int64_t n, uint32_t idmask, const float4* omg,
                      uint32_t* slot_of_id);
int launch_insert_contacts(cudaStream_t st, int64_t m, int64_t n, int64_t stride, uint32_t K,
                           const uint32_t* id_i, const uint32_t* id_j, const float* dt3,
                           const uint32_t* slot_of_id, float4* hist, uint32_t* cnt,
                           uint32_t* flags, int skip_unknown);
int launch_analyze(cudaStream_t st, int64_t n, const StepBuffers& b, const DevGrid& g,
                   unsigned long long* acc);
int launch_max_speed(cudaStream_t st, int64_t n, const float4* vel, uint32_t* out);
int launch_cnt_stats(cudaStream_t st, int64_t n, const uint32_t* cnt,
                     unsigned long long* sum_max);

}  // namespace dem

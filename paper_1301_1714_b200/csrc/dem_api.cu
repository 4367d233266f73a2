// dem_api.cu — host side of libdem.so: the C ABI of include/dem.h.
//
// The host validates, sizes buffers, and enqueues kernels (dem_kernels.cu) on
// the handle's stream, replaying a captured CUDA graph of two steps (one per
// ping-pong parity) so a step costs one graph launch instead of four kernel
// launches. All arithmetic of the method runs in the kernels.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <cstring>
#include <vector>

#include "dem.h"
#include "dem_internal.h"

using namespace dem;

namespace {

struct Alloc {
  void* p;
  size_t bytes;
};

}  // namespace

struct dem_handle {
  dem_params p{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  dem_allocator alloc{};
  bool has_alloc = false;
  std::vector<Alloc> allocs;
  std::string last_error;

  // problem
  int64_t n = -1;  // -1: no particles set yet
  uint32_t K = 16;
  double h = 0.0;
  DevGrid g{};
  DevPhys ph{};
  bool ids_dense = false;
  int64_t id_bound = 0;  // ids < id_bound (slot map size of dem_set_contacts); 0: sparse ids

  // device buffers (ping-pong b in {0,1})
  float4 *pos[2] = {}, *vel[2] = {}, *omg[2] = {};
  uint32_t* key[2] = {};
  float4* hist[2] = {};
  uint32_t* cnt[2] = {};
  uint32_t *prank = nullptr, *count = nullptr, *off = nullptr, *tmp = nullptr, *perm = nullptr;
  float4* pos_sorted = nullptr;
  uint32_t *clist = nullptr, *ccount = nullptr;
  // merge re-sort (single GPU): the integrator's movers,
  // [mover counter, movers this step], movers sorted by (key, slot) and by slot
  uint4* mov = nullptr;      // merge re-sort: two mover lists (by state parity), mov_cap each
  uint32_t* mov_n = nullptr; // their counts
  uint32_t mov_cap = 0;
  bool merge = false;     // merge re-sort in use for this set
  bool merge_ok = false;  // state in the last step's sorted order, movers listed
  bool full_run = false;  // the rest of this dem_step call sorts by counting (mover overflow)
  bool mv_redo = false;   // inside the redo of a mover overflow
  int64_t full_sorts = 0; // steps sorted by the counting sort since dem_set_particles
  uint8_t* cpos = nullptr;
  uint32_t *lcount = nullptr, *llist = nullptr;
  float4* R0 = nullptr;
  float2* R1 = nullptr;
  uint32_t* nslots = nullptr;  // device: input slots of the next step
  uint32_t* flags = nullptr;   // slab mode
  float4 *F = nullptr, *T = nullptr;
  unsigned long long* scan_status[2] = {};
  uint32_t* scan_ctr = nullptr;  // [2]
  uint32_t ntiles = 0;
  DevErr* err = nullptr;
  DevErr* err_host = nullptr;  // pinned
  int64_t cap_n = -1, cap_cells = -1;

  int64_t cap = 0;  // slot capacity = stride of the K-major arrays (single GPU: n)
  float mono_r = 0.f;  // > 0: every particle of the set has this radius (single GPU only)

  // slab decomposition (world_size > 1), DESIGN.md §7
  bool slab = false;
  int rank = 0, world = 1;
  uint8_t* xregion = nullptr;  // this rank's exchange region (cudaMalloc: IPC-shareable)
  XLayout xl{};
  uint64_t xregion_bytes = 0;
  const uint8_t* xleft = nullptr;   // neighbours' regions (peer pointers)
  const uint8_t* xright = nullptr;
  bool xleft_ipc = false, xright_ipc = false;
  bool connected = false;
  uint32_t xbase = 0;  // exchange tag offset of the current set (same sequence on every rank)
  uint32_t nsets = 0;
  XState* xs = nullptr;
  uint32_t* xtiles = nullptr;  // pack tile counts + totals, per state parity [2][xtc_stride]

  int cur = 0;
  int64_t steps = 0;  // completed steps since set_particles (== device step_ctr)
  int fcfg = -1;      // k_force configuration (0 dense, 1 light); -1: chosen at the first step
  float4* mat_tables = nullptr;  // material pair + wall coefficients (cudaMalloc, dem_create)
  float* plate_buf = nullptr;    // plates (R23), 12 floats each (cudaMalloc, dem_create)

  // graphs: g2[b] = two steps starting at parity b; g1[b] = one step
  cudaGraphExec_t g2[2] = {nullptr, nullptr};
  cudaGraphExec_t g1[2] = {nullptr, nullptr};
  // the same with the counting sort (merge mode: the first step, mover overflow)
  cudaGraphExec_t gf2[2] = {nullptr, nullptr};
  cudaGraphExec_t gf1[2] = {nullptr, nullptr};

  // profiling
  bool profiling = false;
  struct Prof {
    cudaEvent_t b, e;
    int kid;
  };
  std::vector<Prof> prof;
  std::vector<cudaEvent_t> event_pool;
  // steps enqueued but not yet checked (DEM_F_ASYNC)
  bool pending = false;
  int64_t pend_ctr0 = 0, pend_steps = 0;
  int pend_cur0 = 0;
  double kernel_ms[8] = {};
  int64_t kernel_count[8] = {};
  int64_t launches = 0, graph_launches = 0;
};

namespace {

thread_local std::string g_tls_error;

int fail(dem_handle* h, int code, const std::string& msg) {
  if (h) h->last_error = msg;
  g_tls_error = msg;
  return code;
}

#define CUDA_TRY(h, call)                                                               \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess)                                                             \
      return fail((h), DEM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

void* dev_alloc(dem_handle* h, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  if (h->has_alloc) {
    p = h->alloc.alloc(h->alloc.ctx, bytes, (void*)h->stream);
  } else {
    if (cudaMallocAsync(&p, bytes, h->stream) != cudaSuccess) p = nullptr;
  }
  if (p) h->allocs.push_back({p, bytes});
  return p;
}

void dev_free(dem_handle* h, void* p) {
  if (!p) return;
  for (size_t i = 0; i < h->allocs.size(); ++i)
    if (h->allocs[i].p == p) {
      if (h->has_alloc)
        h->alloc.free(h->alloc.ctx, p, h->allocs[i].bytes, (void*)h->stream);
      else
        cudaFreeAsync(p, h->stream);
      h->allocs.erase(h->allocs.begin() + (long)i);
      return;
    }
}

template <class T>
bool dalloc(dem_handle* h, T** out, size_t count) {
  *out = (T*)dev_alloc(h, count * sizeof(T));
  return *out != nullptr;
}

void destroy_graphs(dem_handle* h) {
  for (int b = 0; b < 2; ++b) {
    if (h->g2[b]) cudaGraphExecDestroy(h->g2[b]);
    if (h->g1[b]) cudaGraphExecDestroy(h->g1[b]);
    if (h->gf2[b]) cudaGraphExecDestroy(h->gf2[b]);
    if (h->gf1[b]) cudaGraphExecDestroy(h->gf1[b]);
    h->g2[b] = h->g1[b] = h->gf2[b] = h->gf1[b] = nullptr;
  }
}

void free_buffers(dem_handle* h) {
  destroy_graphs(h);
  std::vector<Alloc> all = h->allocs;
  for (auto& a : all) dev_free(h, a.p);
  for (int b = 0; b < 2; ++b) {
    h->pos[b] = h->vel[b] = h->omg[b] = h->hist[b] = nullptr;
    h->key[b] = h->cnt[b] = nullptr;
    h->scan_status[b] = nullptr;
  }
  h->prank = h->count = h->off = h->tmp = h->perm = h->scan_ctr = nullptr;
  h->pos_sorted = nullptr;
  h->clist = h->ccount = h->nslots = h->flags = nullptr;
  h->mov = nullptr;
  h->mov_n = nullptr;
  h->cpos = nullptr;
  h->lcount = h->llist = nullptr;
  h->R0 = nullptr;
  h->R1 = nullptr;
  h->xs = nullptr;
  h->xtiles = nullptr;
  h->F = h->T = nullptr;
  h->err = nullptr;
  h->cap_n = h->cap_cells = -1;
}

StepBuffers step_buffers(dem_handle* h, int b) {
  StepBuffers s{};
  s.pos_in = h->pos[b];
  s.vel_in = h->vel[b];
  s.omg_in = h->omg[b];
  s.pos_out = h->pos[b ^ 1];
  s.vel_out = h->vel[b ^ 1];
  s.omg_out = h->omg[b ^ 1];
  s.key_in = h->key[b];
  s.key_out = h->key[b ^ 1];
  s.prank = h->prank;
  s.count = h->count;
  s.off = h->off;
  s.tmp = h->tmp;
  s.perm = h->perm;
  s.pos_sorted = h->pos_sorted;
  // one radius on the default path (k_detect<MONO> + k_force): the sorted
  // positions carry their old slot in .w, so contact lists hold old slots
  s.sw_r = (h->mono_r > 0.f && !(h->p.flags & (DEM_F_THREAD_PER_PARTICLE | DEM_F_HALF_LISTS)))
               ? h->mono_r : 0.f;
  s.clist = h->clist;
  s.ccount = h->ccount;
  s.nslots = h->nslots;
  s.flags = h->flags;
  s.xtc = h->xtiles ? h->xtiles + (size_t)b * xtc_stride(h->cap) : nullptr;
  s.xtc_next = h->xtiles ? h->xtiles + (size_t)(b ^ 1) * xtc_stride(h->cap) : nullptr;
  s.xntiles = xtc_ntiles(h->cap);
  // slab ranks with a left neighbour: the owned particles' sorted slots start
  // past room for the left ghost plane, which is placed right-aligned below
  s.gl_base = (h->slab && h->rank > 0) ? h->xl.ghost_cap : 0u;
  s.cpos = h->cpos;
  s.lcount = h->lcount;
  s.llist = h->llist;
  s.R0 = h->R0;
  s.R1 = h->R1;
  s.hist_in = h->hist[b];
  s.cnt_in = h->cnt[b];
  s.hist_out = h->hist[b ^ 1];
  s.cnt_out = h->cnt[b ^ 1];
  s.F_out = h->F;
  s.T_out = h->T;
  s.scan_status = h->scan_status[b];
  s.err = h->err;
  if (h->merge) {
    // movers of input parity b (listed by the previous step), and this step's
    s.mv.list_in = h->mov + (size_t)b * h->mov_cap;
    s.mv.n_in = h->mov_n + b;
    s.mv.list_out = h->mov + (size_t)(b ^ 1) * h->mov_cap;
    s.mv.n_out = h->mov_n + (b ^ 1);
    s.mv.cap = h->mov_cap;
  }
  return s;
}

// one radius, dense force configuration: detection runs inside the force
// kernel (k_force<..., FUSED>) unless DEM_F_SPLIT_SWEEP. Measured per
// configuration (profiles/r2_history.md): fused wins where the warps have
// many contact rounds (C3: 0.0894 -> 0.0816 ms/step); on the light bed (C4)
// the split kernels win (0.611 vs 0.631: the detection loop then runs at the
// force kernel's occupancy and L1 share)
#ifndef DEM_FUSED_LIGHT
#define DEM_FUSED_LIGHT 1
#endif
bool fused_sweep(const dem_handle* h) {
  return h->mono_r > 0.f && !(h->p.flags & (DEM_F_THREAD_PER_PARTICLE | DEM_F_HALF_LISTS |
                                            DEM_F_SPLIT_SWEEP)) &&
         (h->fcfg == 0 || (DEM_FUSED_LIGHT && h->fcfg == 1));
}

int kernels_per_step(const dem_handle* h, bool full = false) {
  // counting sort: scan (2) + scatter + rank (+ k_count in merge mode); merge: 2
  const int sort = h->merge ? (full ? 5 : 1) : 4;
  return ((h->p.flags & DEM_F_THREAD_PER_PARTICLE) ? 1 : (h->p.flags & DEM_F_HALF_LISTS) ? 3
          : fused_sweep(h)                         ? 1
                                                   : 2) +
         sort + (h->slab ? (h->merge && !full ? 3 : 4) : 0);
}

// Enqueue one step from parity b: the sort (counting: scan, scatter, rank;
// merge: k_mv_sort, k_mv_perm, k_mv_off), (detect,) sweep. `full`: counting
// sort in merge mode (cell counts from k_count; the integrator lists movers).
// `profile` records an event pair around each kernel.
int enqueue_step(dem_handle* h, int b, bool profile, bool full = false) {
  const StepBuffers s = step_buffers(h, b);
  const bool diag = (h->p.flags & DEM_F_DIAG) != 0;
  cudaEvent_t evb = nullptr;
  auto take = [&]() {
    cudaEvent_t e;
    if (!h->event_pool.empty()) {
      e = h->event_pool.back();
      h->event_pool.pop_back();
    } else {
      cudaEventCreate(&e);
    }
    return e;
  };
  auto rec = [&](int k, bool begin) {
    if (!profile) return;
    cudaEvent_t e = take();
    cudaEventRecord(e, h->stream);
    if (begin) {
      evb = e;
    } else {
      h->prof.push_back({evb, e, k});
    }
  };
  const uint8_t* xl_ = h->xleft ? h->xleft + kXRegionHdr : nullptr;
  const uint8_t* xr_ = h->xright ? h->xright + kXRegionHdr : nullptr;
  if (h->slab) {  // this step's migrants and ghost-plane state from the neighbours (peer memory)
    rec(K_OTHER, true);
    launch_xrecv(h->stream, h->cap, s, h->g, h->K, xl_, xr_, h->xl, h->xs, h->nslots,
                 h->merge && !full);
    rec(K_OTHER, false);
    h->launches += 1;
  }
  if (h->merge && !full) {  // merge re-sort
    rec(K_RANK, true);
    // (slab: the owned particles, their count from the last step's pack)
    launch_merge(h->stream, h->slab ? h->cap : h->n, h->g.ncells, s, h->g,
                 h->slab ? &h->xs->n_out : nullptr, xl_, xr_, h->slab ? &h->xl : nullptr, h->xs);
    rec(K_RANK, false);
    h->launches += 1;
  } else {
    if (h->merge) {  // the integrator listed movers, not cell counts
      rec(K_HASH, true);
      launch_count(h->stream, h->n, s.key_in, h->count, h->prank);
      rec(K_HASH, false);
      cudaMemsetAsync(h->mov_n + (b ^ 1), 0, sizeof(uint32_t), h->stream);  // this step's list
      h->launches += 1;
    }
    rec(K_SCAN, true);
    launch_scan(h->stream, h->count, h->off, h->g.ncells, h->count, s.scan_status, nullptr,
                h->err, 1, s.gl_base);
    rec(K_SCAN, false);
    rec(K_SCATTER, true);
    launch_scatter(h->stream, h->cap, s);
    rec(K_SCATTER, false);
    rec(K_RANK, true);
    launch_rank(h->stream, h->cap, s);
    rec(K_RANK, false);
    h->launches += 4;  // scan is two kernels
  }
  if (h->slab && (full || !h->merge)) {  // (merge steps: blocks of k_merge do it)
    // the neighbours' planes (sorted) and this rank's departed ones: ghost planes
    rec(K_OTHER, true);
    launch_xghost_place(h->stream, h->cap, s, h->g, xl_, xr_, h->xl, h->xs);
    rec(K_OTHER, false);
    h->launches += 1;
  }
  // default: full contact lists (k_detect + warp-flattened k_force); the half
  // lists (Newton's third law) and the paper's fused mapping are ablations
  // one radius, dense/light: detection fused into the force kernel unless
  // DEM_F_SPLIT_SWEEP (6: fused dense, 7: fused light)
  const bool fused = fused_sweep(h);
  const int variant = (h->p.flags & DEM_F_THREAD_PER_PARTICLE) ? 1
                      : (h->p.flags & DEM_F_HALF_LISTS)        ? 0
                      : (h->fcfg == 3)                         ? 5
                      : (h->fcfg == 2)                         ? 4
                      : fused                                  ? (h->fcfg == 1 ? 7 : 6)
                      : (h->fcfg == 1)                         ? 3
                                                               : 2;
  if (variant == 0) {  // half lists: detect, pair, finish
    rec(K_DETECT, true);
    launch_detect_half(h->stream, h->cap, h->K, s, h->g);
    rec(K_DETECT, false);
    rec(K_SWEEP, true);
    launch_pair(h->stream, h->cap, h->K, h->p.model, s, h->g, h->ph);
    rec(K_SWEEP, false);
    rec(K_FINISH, true);
    launch_finish(h->stream, h->cap, h->K, h->p.model, diag, s, h->g, h->ph);
    rec(K_FINISH, false);
    h->launches += 2;
  } else {
    if (variant >= 2 && variant < 6) {
      rec(K_DETECT, true);
      launch_detect(h->stream, h->cap, h->K, s, h->g, h->mono_r, variant >= 3);
      rec(K_DETECT, false);
      h->launches += 1;
    }
    rec(K_SWEEP, true);
    launch_sweep(h->stream, h->cap, h->K, h->p.model, diag, s, h->g, h->ph, variant);
    rec(K_SWEEP, false);
  }
  h->launches += 1;
  if (h->slab) {  // pack and publish the next step's boundary planes and migrants
    rec(K_OTHER, true);
    launch_xpack(h->stream, h->cap, s, h->g, h->K, h->xregion + kXRegionHdr, h->xl, h->xs, 0,
                 (h->rank > 0 ? 1 : 0) | (h->rank < h->world - 1 ? 2 : 0));
    rec(K_OTHER, false);
    h->launches += 2;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, DEM_ECUDA, std::string("step launch: ") + cudaGetErrorString(e));
  return DEM_OK;
}

int build_graph(dem_handle* h, int b, int nsteps, cudaGraphExec_t* out, bool full = false) {
  cudaGraph_t graph;
  CUDA_TRY(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int parity = b;
  int64_t l0 = h->launches;
  for (int k = 0; k < nsteps; ++k) {
    enqueue_step(h, parity, false, full);
    parity ^= 1;
  }
  h->launches = l0;
  CUDA_TRY(h, cudaStreamEndCapture(h->stream, &graph));
  cudaError_t e = cudaGraphInstantiate(out, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(h, DEM_ECUDA, std::string("graph: ") + cudaGetErrorString(e));
  return DEM_OK;
}

const char* err_name(uint32_t code) {
  switch (code) {
    case 6: return "contact history capacity (max_contacts) exceeded";
    case 7: return "non-finite state (explosion)";
    case 8: return "particle escaped through a wall";
    case 9: return "coincident centres in contact";
    default: return "unknown";
  }
}

// Wait for the stream and turn a device error record into a return code,
// rolling the state back to the last completed step.
int check_step_error(dem_handle* h, int64_t ctr0, int cur0, int64_t nsteps) {
  CUDA_TRY(h, cudaMemcpyAsync(h->err_host, h->err, sizeof(DevErr), cudaMemcpyDeviceToHost,
                              h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  const DevErr e = *h->err_host;
  if (e.code == 0) {
    h->steps = ctr0 + nsteps;
    if (h->slab) {  // particles this rank advanced in its last step
      XState x{};
      CUDA_TRY(h, cudaMemcpy(&x, h->xs, sizeof x, cudaMemcpyDeviceToHost));
      h->n = x.n_out;
    }
    return DEM_OK;
  }
  if (h->slab) {  // no roll-back across ranks: the handle must be set again
    char buf[240];
    if (e.code == 11u && e.slot == 0xFFFFFE00u)
      snprintf(buf, sizeof buf,
               "slab exchange failed (slab rank %d): a neighbour's step failed (its publication "
               "is poisoned) before step %u; set the particles again on every rank",
               h->rank, e.step);
    else if (e.code == 11u && (e.slot & 0xFFFFFF00u) == 0xFFFFFF00u)
      snprintf(buf, sizeof buf,
               "slab exchange failed (slab rank %d): neighbour publication of tag %u never "
               "arrived (seen: left %u, right %u, low bits) in step %u; set the particles again",
               h->rank, e.slot & 0xFFu, e.id >> 16, e.id & 0xFFFFu, e.step);
    else
      snprintf(buf, sizeof buf, "%s (slab rank %d): particle id %u in step %u; set the particles again",
               e.code == 11u ? "slab exchange failed (a migrant skipped a plane)"
                             : err_name(e.code),
               h->rank, e.id, e.step);
    h->n = -1;
    return fail(h, e.code == 11u ? DEM_EPEER : -(int)e.code, buf);
  }
  const int64_t failed = (int64_t)e.step;  // 1-based counter value of the failing step
  const int64_t done = std::max<int64_t>(0, failed - 1 - ctr0);
  h->cur = cur0 ^ (int)(done & 1);
  h->steps = ctr0 + done;
  // restore the per-step scratch for the good state and clear the record
  CUDA_TRY(h, cudaMemsetAsync(h->count, 0, sizeof(uint32_t) * h->g.ncells, h->stream));
  // counting sort: the cell counts of the good state; merge mode: the next
  // step sorts by counting (its k_count counts) since the failed step may have
  // updated the offsets, SCM and mover list in place
  if (h->merge) {
    h->merge_ok = false;
    CUDA_TRY(h, cudaMemsetAsync(h->mov_n, 0, 2 * sizeof(uint32_t), h->stream));
  } else {
    launch_count(h->stream, h->n, h->key[h->cur], h->count, h->prank);
  }
  CUDA_TRY(h, cudaMemsetAsync(h->scan_status[0], 0, sizeof(unsigned long long) * h->ntiles,
                              h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->scan_status[1], 0, sizeof(unsigned long long) * h->ntiles,
                              h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->scan_ctr, 0, 2 * sizeof(uint32_t), h->stream));
  DevErr clean{};
  clean.step_ctr = (uint32_t)h->steps;
  CUDA_TRY(h, cudaMemcpyAsync(h->err, &clean, sizeof(DevErr), cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (e.code == 12u) {
    // more movers than the merge re-sort takes: that step is redone by
    // counting (merge_ok is false) and the next ones merge again; a second
    // overflow inside the redo sorts the rest of the call by counting
    const int64_t left = nsteps - done;
    const bool again = h->mv_redo;
    h->mv_redo = true;
    h->full_run = again;
    int rc = dem_step(h, left);
    h->full_run = false;
    h->mv_redo = again;
    if (rc) return rc;
    return dem_sync(h);
  }
  int code = -(int)e.code;
  char buf[256];
  snprintf(buf, sizeof buf, "%s: particle id %u (slot %u) in step %lld; state kept at step %lld",
           err_name(e.code), e.id, e.slot, (long long)failed, (long long)h->steps);
  return fail(h, code, buf);
}

int validate_params(const dem_params* p) {
  if (!p) return DEM_EINVAL;
  if (p->abi_version != DEM_ABI_VERSION) return DEM_EABI;
  if (p->model != DEM_MODEL_PRACTICAL && p->model != DEM_MODEL_SIMPLE) return DEM_EINVAL;
  if (!(p->dt > 0.0f) || !std::isfinite(p->dt)) return DEM_EINVAL;
  for (int a = 0; a < 3; ++a)
    if (!(p->box_hi[a] > p->box_lo[a]) || !std::isfinite(p->box_lo[a]) ||
        !std::isfinite(p->box_hi[a]) || !std::isfinite(p->gravity[a]))
      return DEM_EINVAL;
  const float nonneg[] = {p->stiffness_n, p->stiffness_t, p->damping, p->friction,
                          p->k_sp, p->k_da, p->k_sh};
  for (float v : nonneg)
    if (!(v >= 0.0f) || !std::isfinite(v)) return DEM_EINVAL;
  if (p->cell_edge < 0.0f || !std::isfinite(p->cell_edge)) return DEM_EINVAL;
  // list capacity K: at most kMaxContacts (a warp's contacts are indexed in
  // 16 bits, list indices in a byte); the half-list ablation packs its lower
  // lists as (slot << 5 | index), so it needs K <= 32
  if (p->max_contacts > kMaxContacts) return DEM_EINVAL;
  if ((p->flags & DEM_F_HALF_LISTS) && p->max_contacts > 32) return DEM_EINVAL;
  // the ablations live in libdem_ablations.so
  if ((p->flags & (DEM_F_THREAD_PER_PARTICLE | DEM_F_HALF_LISTS | DEM_F_FORCE_LANES | DEM_F_FORCE_WS)) &&
      !ablations_built())
    return DEM_EINVAL;
  if (p->world_size > 1 && (p->rank < 0 || p->rank >= p->world_size)) return DEM_EINVAL;
  if (p->n_plates > 10 || (p->n_plates && !p->plates)) return DEM_EINVAL;
  for (uint32_t k = 0; k < p->n_plates; ++k) {  // unit normal, unit axis in the plane, extents
    const float* q = p->plates + 12 * k;
    for (int c = 0; c < 11; ++c)
      if (!std::isfinite(q[c])) return DEM_EINVAL;
    const double nn = (double)q[3] * q[3] + (double)q[4] * q[4] + (double)q[5] * q[5];
    const double uu = (double)q[6] * q[6] + (double)q[7] * q[7] + (double)q[8] * q[8];
    const double nu = (double)q[3] * q[6] + (double)q[4] * q[7] + (double)q[5] * q[8];
    if (std::fabs(nn - 1) > 1e-5 || std::fabs(uu - 1) > 1e-5 || std::fabs(nu) > 1e-5 ||
        !(q[9] > 0.f) || !(q[10] > 0.f))
      return DEM_EINVAL;
  }
  if (p->n_materials > 1) {  // symmetric, finite, non-negative (SPEC MaterialTable)
    const uint32_t M = p->n_materials;
    if (M > 16 || !p->material_pairs) return DEM_EINVAL;
    for (uint32_t i = 0; i < M; ++i)
      for (uint32_t j = 0; j < M; ++j)
        for (int c = 0; c < 4; ++c) {
          const float v = p->material_pairs[((size_t)i * M + j) * 4 + c];
          if (!(v >= 0.0f) || !std::isfinite(v) ||
              v != p->material_pairs[((size_t)j * M + i) * 4 + c])
            return DEM_EINVAL;
        }
    if (p->material_walls)
      for (uint32_t k = 0; k < 4 * M; ++k)
        if (!(p->material_walls[k] >= 0.0f) || !std::isfinite(p->material_walls[k]))
          return DEM_EINVAL;
  }
  return DEM_OK;
}

}  // namespace

extern "C" {

const char* dem_strerror(int code) {
  switch (code) {
    case DEM_OK: return "ok";
    case DEM_EINVAL: return "invalid argument";
    case DEM_EABI: return "ABI version mismatch";
    case DEM_ENOMEM: return "out of device memory";
    case DEM_ECUDA: return "CUDA error";
    case DEM_ENCCL: return "NCCL error";
    case DEM_EOVERFLOW: return "contact history capacity exceeded";
    case DEM_ENONFINITE: return "non-finite particle state";
    case DEM_EESCAPED: return "particle escaped through a wall";
    case DEM_ECOINCIDENT: return "coincident particle centres";
    case DEM_ESTATE: return "call out of order";
    default: return "unknown error";
  }
}

const char* dem_last_error(const dem_handle* h) {
  return h ? h->last_error.c_str() : g_tls_error.c_str();
}

int dem_create(const dem_params* p, dem_handle** out) {
  if (!out) return DEM_EINVAL;
  *out = nullptr;
  int rc = validate_params(p);
  if (rc != DEM_OK) return fail(nullptr, rc, "dem_create: invalid params");
  dem_handle* h = new dem_handle();
  h->p = *p;
  h->K = p->max_contacts ? p->max_contacts : 16u;
  h->slab = p->world_size > 1;
  h->rank = h->slab ? p->rank : 0;
  h->world = h->slab ? p->world_size : 1;
  if (p->device >= 0) {
    if (cudaSetDevice(p->device) != cudaSuccess) {
      delete h;
      return fail(nullptr, DEM_ECUDA, "cudaSetDevice failed");
    }
  }
  if (cudaGetDevice(&h->device) != cudaSuccess) {
    delete h;
    return fail(nullptr, DEM_ECUDA, "no CUDA device");
  }
  if (p->stream) {
    h->stream = (cudaStream_t)p->stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete h;
      return fail(nullptr, DEM_ECUDA, "cudaStreamCreate failed");
    }
    h->own_stream = true;
  }
  if (p->allocator) {
    h->alloc = *p->allocator;
    h->has_alloc = h->alloc.alloc && h->alloc.free;
  }
  if (cudaMallocHost((void**)&h->err_host, sizeof(DevErr)) != cudaSuccess) {
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
    return fail(nullptr, DEM_ENOMEM, "pinned allocation failed");
  }
  // physics constants (fp32 as given; wall values < 0 fall back to the particle's)
  DevPhys& ph = h->ph;
  ph.dt = p->dt;
  for (int a = 0; a < 3; ++a) ph.g[a] = p->gravity[a];
  ph.Cn = p->stiffness_n;
  ph.Ct = p->stiffness_t;
  ph.alpha = p->damping;
  ph.mu = p->friction;
  ph.wCn = p->wall_stiffness_n >= 0 ? p->wall_stiffness_n : p->stiffness_n;
  ph.wCt = p->wall_stiffness_t >= 0 ? p->wall_stiffness_t : p->stiffness_t;
  ph.walpha = p->wall_damping >= 0 ? p->wall_damping : p->damping;
  ph.wmu = p->wall_friction >= 0 ? p->wall_friction : p->friction;
  ph.ksp = p->k_sp;
  ph.kda = p->k_da;
  ph.ksh = p->k_sh;
  ph.flags = p->flags & (DEM_F_TRUNCATE_DT | DEM_F_CLAMP_FN);
  // material pairs (Eqs. 5, 8-10 as functions of (i, j)): device tables
  ph.nmat = 1;
  ph.idmask = 0xFFFFFFFFu;
  if (p->n_materials > 1) {
    const uint32_t M = p->n_materials;
    std::vector<float4> t((size_t)M * M), w(M);
    for (uint32_t i = 0; i < M; ++i) {
      for (uint32_t j = 0; j < M; ++j) {
        const float* c = p->material_pairs + ((size_t)i * M + j) * 4;
        t[(size_t)i * M + j] = make_float4(c[0], c[1], c[2], c[3]);
      }
      if (p->material_walls) {
        const float* c = p->material_walls + (size_t)i * 4;
        w[i] = make_float4(c[0], c[1], c[2], c[3]);
      } else {
        w[i] = make_float4(ph.wCn, ph.wCt, ph.walpha, ph.wmu);
      }
    }
    if (cudaMalloc((void**)&h->mat_tables, sizeof(float4) * (t.size() + w.size())) != cudaSuccess ||
        cudaMemcpy(h->mat_tables, t.data(), sizeof(float4) * t.size(), cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMemcpy(h->mat_tables + t.size(), w.data(), sizeof(float4) * w.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess) {
      if (h->mat_tables) cudaFree(h->mat_tables);
      cudaFreeHost(h->err_host);
      if (h->own_stream) cudaStreamDestroy(h->stream);
      delete h;
      return fail(nullptr, DEM_ENOMEM, "material table allocation failed");
    }
    ph.nmat = M;
    ph.mat = h->mat_tables;
    ph.wmat = h->mat_tables + t.size();
    ph.idmask = (1u << kMatShift) - 1u;
  }
  ph.nplates = 0;
  ph.plates = nullptr;
  if (p->n_plates) {
    if (cudaMalloc((void**)&h->plate_buf, sizeof(float) * 12 * p->n_plates) != cudaSuccess ||
        cudaMemcpy(h->plate_buf, p->plates, sizeof(float) * 12 * p->n_plates,
                   cudaMemcpyHostToDevice) != cudaSuccess) {
      if (h->plate_buf) cudaFree(h->plate_buf);
      if (h->mat_tables) cudaFree(h->mat_tables);
      cudaFreeHost(h->err_host);
      if (h->own_stream) cudaStreamDestroy(h->stream);
      delete h;
      return fail(nullptr, DEM_ENOMEM, "plate allocation failed");
    }
    ph.plates = h->plate_buf;
    ph.nplates = p->n_plates;
  }
  *out = h;
  return DEM_OK;
}

int dem_destroy(dem_handle* h) {
  if (!h) return DEM_OK;
  cudaStreamSynchronize(h->stream);
  if (h->xleft_ipc && h->xleft) cudaIpcCloseMemHandle((void*)h->xleft);
  if (h->xright_ipc && h->xright) cudaIpcCloseMemHandle((void*)h->xright);
  if (h->xregion) cudaFree(h->xregion);
  if (h->mat_tables) cudaFree(h->mat_tables);
  if (h->plate_buf) cudaFree(h->plate_buf);
  free_buffers(h);
  for (auto& pr : h->prof) {
    cudaEventDestroy(pr.b);
    cudaEventDestroy(pr.e);
  }
  for (auto e : h->event_pool) cudaEventDestroy(e);
  cudaStreamSynchronize(h->stream);
  if (h->err_host) cudaFreeHost(h->err_host);
  if (h->own_stream) cudaStreamDestroy(h->stream);
  delete h;
  return DEM_OK;
}

int dem_set_particles(dem_handle* h, int64_t n, const dem_particles* src) {
  if (!h) return DEM_EINVAL;
  if (n < 0 || n > 0x7FFFFFF0LL || (n > 0 && (!src || !src->pos)))
    return fail(h, DEM_EINVAL, "dem_set_particles: bad n or NULL pos");
  cudaStream_t st = h->stream;
  // 1. stage inputs on the device
  PackIn in{};
  std::vector<void*> staged;
  auto stage = [&](const void* p, size_t bytes) -> const void* {
    if (!p) return nullptr;
    if (src->mem_kind == DEM_MEM_DEVICE) return p;
    void* d = dev_alloc(h, bytes);
    if (!d) return nullptr;
    staged.push_back(d);
    cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, st);
    return d;
  };
  if (src && src->mem_kind == DEM_MEM_DEVICE && !h->own_stream) cudaStreamSynchronize(nullptr);
  const size_t n3 = (size_t)n * 3 * sizeof(float), n1 = (size_t)n * sizeof(float);
  in.pos = n ? (const float*)stage(src->pos, n3) : nullptr;
  in.vel = n ? (const float*)stage(src->vel, n3) : nullptr;
  in.omega = n ? (const float*)stage(src->omega, n3) : nullptr;
  in.radius = n ? (const float*)stage(src->radius, n1) : nullptr;
  in.mass = n ? (const float*)stage(src->mass, n1) : nullptr;
  in.id = n ? (const uint32_t*)stage(src->id, (size_t)n * 4) : nullptr;
  in.material = n && h->ph.nmat > 1 ? (const uint32_t*)stage(src->material, (size_t)n * 4) : nullptr;
  in.nmat = h->ph.nmat;
  in.def_radius = h->p.radius;
  in.def_mass_coef = (float)(h->p.density * (4.0 / 3.0) * M_PI);
  auto unstage = [&]() {
    for (void* d : staged) dev_free(h, d);
  };
  if (n && !in.pos) {
    unstage();
    return fail(h, DEM_ENOMEM, "staging allocation failed");
  }
  // 2. probe: validity, r_max, id_max
  Probe* probe = nullptr;
  if (!dalloc(h, &probe, 1)) {
    unstage();
    return fail(h, DEM_ENOMEM, "probe allocation failed");
  }
  DevGrid g{};
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = (double)h->p.box_lo[a];
    g.hi[a] = (double)h->p.box_hi[a];
  }
  CUDA_TRY(h, cudaMemsetAsync(probe, 0, sizeof(Probe), st));
  launch_probe(st, n, in, g, probe);
  Probe hp{};
  CUDA_TRY(h, cudaMemcpyAsync(&hp, probe, sizeof(Probe), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  dev_free(h, probe);
  if (hp.bad_radius || hp.bad_mass || hp.nonfinite || hp.outside || hp.bad_id ||
      hp.bad_material) {
    unstage();
    char buf[240];
    snprintf(buf, sizeof buf,
             "dem_set_particles: %u bad radii, %u bad masses, %u non-finite, %u outside the "
             "box, %u ids >= %s, %u materials >= n_materials",
             hp.bad_radius, hp.bad_mass, hp.nonfinite, hp.outside, hp.bad_id,
             h->ph.nmat > 1 ? "2^27 (materials in use)" : "0xFFFFFFF0", hp.bad_material);
    return fail(h, DEM_EINVAL, buf);
  }
  // 3. the CDG (R15): h = cell_edge or 2 r_max (1 + 2^-10); n_a = floor(L_a / h) >= 3
  float rmax = 0.f, rmin = 0.f;
  memcpy(&rmax, &hp.rmax_bits, 4);
  const uint32_t rmin_bits = ~hp.rmin_cbits;
  memcpy(&rmin, &rmin_bits, 4);
  // one radius: the candidate test's S² is a constant and the sorted
  // positions carry old slots. Slab ranks are each given the whole set, so
  // they all see the same radii; dem_connect refuses a neighbour whose set
  // said otherwise (XLayout::mono_bits)
  h->mono_r = (n > 0 && rmin == rmax && !(h->p.flags & DEM_F_GENERAL_DETECT)) ? rmax : 0.f;
  const double hmin = 2.0 * (double)rmax * (1.0 + std::ldexp(1.0, -10));
  double hc = h->p.cell_edge > 0.0f ? (double)h->p.cell_edge : hmin;
  if (hc < hmin || !(hc > 0.0)) {
    unstage();
    return fail(h, DEM_EINVAL, "cell edge smaller than 2 r_max (1 + 2^-10)");
  }
  int64_t dims[3];
  for (int a = 0; a < 3; ++a) {
    double q = std::floor((g.hi[a] - g.lo[a]) / hc);
    if (!(q >= 3.0) || q > 1e9) {
      unstage();
      return fail(h, DEM_EINVAL, "grid dimension < 3 (box too small for the cell edge)");
    }
    dims[a] = (int64_t)q;
  }
  const int64_t ncells = dims[0] * dims[1] * dims[2];
  if (ncells >= (int64_t)0xFFFFFFF0LL) {
    unstage();
    return fail(h, DEM_EINVAL, "too many grid cells (> 2^32)");
  }
  g.nx = (int)dims[0];
  g.ny = (int)dims[1];
  g.nz = (int)dims[2];
  g.ncells = (uint32_t)ncells;
  g.inv_h = 1.0 / hc;
  g.nz_global = g.nz;
  g.zlo = 0;
  g.z0 = 0;
  g.z1 = g.nz;
  g.own_c0 = 0;
  g.own_c1 = g.ncells;
  g.trash = g.ncells;
  g.slab = 0;
  int64_t n_own = n;    // particles this rank keeps
  int64_t cap = n;      // slot capacity
  uint32_t *keep = nullptr, *dst = nullptr;
  if (h->slab) {
    // 3b. slabs along z (the slowest axis of the cell index): rank r owns the
    // planes [z0, z1); its local grid adds one ghost plane on each side
    const int P = h->world, r = h->rank;
    const int z0 = (int)((int64_t)r * g.nz_global / P), z1 = (int)((int64_t)(r + 1) * g.nz_global / P);
    if (z1 - z0 < 2) {
      unstage();
      return fail(h, DEM_EINVAL, "slab thinner than 2 cell planes: fewer ranks or smaller cells");
    }
    g.z0 = z0;
    g.z1 = z1;
    g.zlo = std::max(z0 - 1, 0);
    const int zhi = std::min(z1 + 1, g.nz_global);
    g.nz = zhi - g.zlo;
    const uint32_t plane = (uint32_t)g.nx * (uint32_t)g.ny;
    g.trash = plane * (uint32_t)g.nz;
    g.ncells = g.trash + 1u;  // + the trash cell that collects departed particles
    g.own_c0 = (uint32_t)(z0 - g.zlo) * plane;
    g.own_c1 = (uint32_t)(z1 - g.zlo) * plane;
    g.slab = 1;
    // tags continue across re-sets, so a neighbour never mistakes an old
    // publication for the new one (every rank runs the same set/step sequence)
    if (h->nsets++ > 0) h->xbase += (uint32_t)h->steps + 2u;
    g.xbase = h->xbase;
    // this rank's particles, compacted in input order (deterministic)
    unsigned long long* st_tiles = nullptr;
    uint32_t* ctr = nullptr;
    const uint32_t kt = (uint32_t)((n + kScanTile - 1) / kScanTile) + 1;
    if (!dalloc(h, &keep, (size_t)std::max<int64_t>(n, 1)) ||
        !dalloc(h, &dst, (size_t)std::max<int64_t>(n, 1) + 1) || !dalloc(h, &st_tiles, kt) ||
        !dalloc(h, &ctr, 1)) {
      unstage();
      return fail(h, DEM_ENOMEM, "allocation failed");
    }
    launch_keep(st, n, in.pos, g, keep);
    launch_scan(st, keep, dst, (uint32_t)n, nullptr, st_tiles, ctr, nullptr, 0);
    uint32_t kept = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&kept, dst + n, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    dev_free(h, st_tiles);
    dev_free(h, ctr);
    n_own = kept;
    // exchange capacities from the most populated z-plane of the whole input
    // set, so that every rank given the same set builds the same layout (a
    // neighbour reads this rank's blocks at its own offsets; checked at connect)
    uint32_t* ph = nullptr;
    if (!dalloc(h, &ph, (size_t)g.nz_global)) {
      unstage();
      return fail(h, DEM_ENOMEM, "allocation failed");
    }
    CUDA_TRY(h, cudaMemsetAsync(ph, 0, sizeof(uint32_t) * g.nz_global, st));
    launch_plane_hist(st, n, in.pos, g, ph);
    std::vector<uint32_t> hh((size_t)g.nz_global);
    CUDA_TRY(h, cudaMemcpyAsync(hh.data(), ph, sizeof(uint32_t) * g.nz_global, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    dev_free(h, ph);
    const int64_t per_plane = (int64_t)*std::max_element(hh.begin(), hh.end()) + 1;
    const uint32_t gcap = (uint32_t)std::max<int64_t>(4096, 2 * per_plane + 1024);
    const uint32_t mcap = std::max<uint32_t>(1024, gcap / 4);
    cap = n_own + n_own / 4 + 2 * (int64_t)gcap + 2 * (int64_t)mcap;
    h->xl = XLayout::make(mcap, gcap, h->K, plane);
    memcpy(&h->xl.mono_bits, &h->mono_r, 4);
  }
  const int64_t ncl = g.ncells;  // cells the scan covers (local + trash in slab mode)
  // 4. buffers (reallocated when the capacity or the grid changes)
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (h->cap_n != cap || h->cap_cells != ncl) {
    // keep staged inputs alive: free only the persistent buffers
    std::vector<void*> keepalive(staged);
    keepalive.push_back(keep);
    keepalive.push_back(dst);
    destroy_graphs(h);
    std::vector<Alloc> all = h->allocs;
    for (auto& a : all)
      if (std::find(keepalive.begin(), keepalive.end(), a.p) == keepalive.end()) dev_free(h, a.p);
    const size_t N = (size_t)(cap > 0 ? cap : 1);
    const int64_t ncells = ncl;
    const uint32_t ntiles = (uint32_t)((std::max<int64_t>(ncells, cap) + kScanTile - 1) / kScanTile) + 1;
    bool ok = true;
    for (int b = 0; b < 2; ++b) {
      ok &= dalloc(h, &h->pos[b], N) && dalloc(h, &h->vel[b], N) && dalloc(h, &h->omg[b], N) &&
            dalloc(h, &h->key[b], N) && dalloc(h, &h->cnt[b], N) &&
            dalloc(h, &h->hist[b], N * h->K) && dalloc(h, &h->scan_status[b], ntiles);
    }
    ok &= dalloc(h, &h->prank, N) && dalloc(h, &h->count, (size_t)ncells + 1) &&
          dalloc(h, &h->off, (size_t)ncells + 1) && dalloc(h, &h->tmp, N) &&
          dalloc(h, &h->perm, N) && dalloc(h, &h->pos_sorted, N) && dalloc(h, &h->clist, N * h->K) &&
          dalloc(h, &h->ccount, N) && dalloc(h, &h->nslots, 1) && dalloc(h, &h->scan_ctr, 2) &&
          dalloc(h, &h->err, 1);
    if (h->p.flags & DEM_F_DIAG) ok &= dalloc(h, &h->F, N) && dalloc(h, &h->T, N);
    if (h->p.flags & DEM_F_HALF_LISTS)
      ok &= dalloc(h, &h->cpos, N * h->K) && dalloc(h, &h->lcount, N) &&
            dalloc(h, &h->llist, N * h->K) && dalloc(h, &h->R0, N * h->K) &&
            dalloc(h, &h->R1, N * h->K);
    // merge re-sort buffers (slab ranks: room for the arriving migrants too)
    const uint32_t mvc = mover_cap(cap) + (h->slab ? 2 * h->xl.mig_cap : 0u);
    ok &= dalloc(h, &h->mov, 2 * (size_t)mvc) && dalloc(h, &h->mov_n, 2);
    h->mov_cap = mvc;
    if (h->slab) {
      ok &= dalloc(h, &h->flags, N) && dalloc(h, &h->xs, 1) &&
            dalloc(h, &h->xtiles, 2 * (size_t)xtc_stride(N));
    }
    // defined contents everywhere (once per allocation): several kernels load
    // ahead of their bounds checks (entries past a count, slots past nslots)
    // and discard the values; this keeps compute-sanitizer's initcheck clean
    if (ok) {
      std::vector<Alloc> fresh = h->allocs;
      for (auto& a : fresh)
        if (std::find(keepalive.begin(), keepalive.end(), a.p) == keepalive.end())
          ok &= cudaMemsetAsync(a.p, 0, a.bytes, st) == cudaSuccess;
    }
    if (!ok) {
      unstage();
      free_buffers(h);
      h->n = -1;
      return fail(h, DEM_ENOMEM, "device allocation failed");
    }
    h->ntiles = ntiles;
    h->cap_n = cap;
    h->cap_cells = ncl;
  }
  if (h->slab) {  // exchange region: (re)allocated when the layout needs more room
    const uint64_t need = kXRegionHdr + 4 * h->xl.bytes;
    if (!h->xregion || h->xregion_bytes < need) {
      if (h->xregion) cudaFree(h->xregion);
      h->xregion = nullptr;
      h->xregion_bytes = 0;
      h->connected = false;  // the neighbours must reconnect to the new region
      if (cudaMalloc((void**)&h->xregion, need) != cudaSuccess) {
        unstage();
        h->n = -1;
        return fail(h, DEM_ENOMEM, "exchange region allocation failed");
      }
      CUDA_TRY(h, cudaMemset(h->xregion, 0, need));
      h->xregion_bytes = need;
    }
    CUDA_TRY(h, cudaMemcpy(h->xregion, &h->xl, sizeof(XLayout), cudaMemcpyHostToDevice));
  }
  h->g = g;
  h->h = hc;
  h->n = n_own;
  h->cap = cap;
  h->cur = 0;
  h->steps = 0;
  h->fcfg = -1;
  destroy_graphs(h);
  const size_t N = (size_t)(cap > 0 ? cap : 1);
  const int64_t ncells_a = ncl;
  CUDA_TRY(h, cudaMemsetAsync(h->count, 0, sizeof(uint32_t) * ((size_t)ncells_a + 1), st));
  CUDA_TRY(h, cudaMemsetAsync(h->off, 0, sizeof(uint32_t) * ((size_t)ncells_a + 1), st));
  CUDA_TRY(h, cudaMemsetAsync(h->perm, 0, sizeof(uint32_t) * N, st));
  // k_force reads the first 4 list entries before the count arrives (unused
  // beyond it); defined contents keep compute-sanitizer's initcheck clean
  CUDA_TRY(h, cudaMemsetAsync(h->clist, 0, sizeof(uint32_t) * N * h->K, st));
  CUDA_TRY(h, cudaMemsetAsync(h->cnt[0], 0, sizeof(uint32_t) * N, st));
  CUDA_TRY(h, cudaMemsetAsync(h->cnt[1], 0, sizeof(uint32_t) * N, st));
  for (int b = 0; b < 2; ++b)
    CUDA_TRY(h, cudaMemsetAsync(h->scan_status[b], 0, sizeof(unsigned long long) * h->ntiles, st));
  CUDA_TRY(h, cudaMemsetAsync(h->scan_ctr, 0, 2 * sizeof(uint32_t), st));
  CUDA_TRY(h, cudaMemsetAsync(h->err, 0, sizeof(DevErr), st));
  {
    const uint32_t nn = (uint32_t)n_own;
    CUDA_TRY(h, cudaMemcpyAsync(h->nslots, &nn, 4, cudaMemcpyHostToDevice, st));
    if (h->slab) {
      XState x{};
      x.n_out = nn;
      CUDA_TRY(h, cudaMemcpyAsync(h->xs, &x, sizeof x, cudaMemcpyHostToDevice, st));
    }
    CUDA_TRY(h, cudaStreamSynchronize(st));
  }
  if (h->F) CUDA_TRY(h, cudaMemsetAsync(h->F, 0, sizeof(float4) * N, st));
  if (h->T) CUDA_TRY(h, cudaMemsetAsync(h->T, 0, sizeof(float4) * N, st));
  // 5. pack + hash (step 2 for the first step) + counting ranks
  launch_pack(st, n, in, g, h->pos[0], h->vel[0], h->omg[0], h->key[0], h->count, h->prank, dst,
              keep);
  h->launches += (n > 0) ? 2 : 1;
  // merge re-sort (single GPU unless DEM_F_FULL_SORT): the first step sorts by
  // counting with its own k_count, so the cell counts start from zero
  // (slab ranks always merge: a departed migrant is a removal of the merge and
  // joins this rank's ghost plane in k_xghost_place)
  h->merge = h->slab || !(h->p.flags & DEM_F_FULL_SORT);
  h->merge_ok = h->full_run = false;
  h->full_sorts = 0;
  if (h->merge && !h->slab) {
    CUDA_TRY(h, cudaMemsetAsync(h->count, 0, sizeof(uint32_t) * ((size_t)ncells_a + 1), st));
    CUDA_TRY(h, cudaMemsetAsync(h->mov_n, 0, 2 * sizeof(uint32_t), st));
  }
  sweep_prepare(h->K);
  if (h->slab) {
    // 5b. publish the set state's boundary planes (sorted) for the neighbours'
    // first step: a counting sort of the owned particles (k_pack counted
    // them) into pos_sorted from gl_base, then the planes' sorted runs
    dev_free(h, keep);
    dev_free(h, dst);
    launch_flags(st, n_own, h->pos[0], g, h->flags);
    StepBuffers sb = step_buffers(h, 0);
    launch_scan(st, h->count, h->off, g.ncells, h->count, sb.scan_status, nullptr, h->err, 0,
                sb.gl_base);
    launch_scatter(st, cap, sb);
    launch_rank(st, cap, sb);
    sb.pos_out = h->pos[0];  // (the set state: the planes' state is read through the old slot)
    sb.vel_out = h->vel[0];
    sb.omg_out = h->omg[0];
    sb.cnt_out = h->cnt[0];
    sb.hist_out = h->hist[0];
    // the first step (state parity 0) accumulates into parity 0's counts:
    // the set state's counts take parity 1's, and everything starts at zero
    CUDA_TRY(h, cudaMemsetAsync(h->xtiles, 0, 2 * sizeof(uint32_t) * xtc_stride(cap), st));
    sb.xtc = h->xtiles + xtc_stride(cap);
    sb.xtc_next = h->xtiles;
    launch_xpack(st, cap, sb, g, h->K, h->xregion + kXRegionHdr, h->xl, h->xs, 1,
                 (h->rank > 0 ? 1 : 0) | (h->rank < h->world - 1 ? 2 : 0));
    // the first step sorts by counting again (k_count); the scan zeroed the counts
    CUDA_TRY(h, cudaMemsetAsync(h->mov_n, 0, 2 * sizeof(uint32_t), st));
    DevErr e{};
    CUDA_TRY(h, cudaMemcpyAsync(&e, h->err, sizeof e, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    unstage();
    if (e.code != 0u) {
      h->n = -1;
      char buf[200];
      snprintf(buf, sizeof buf,
               "dem_set_particles: publishing the boundary planes for the neighbours failed "
               "(%s at output slot %u, particle id %u; ghost capacity %u, migrant capacity %u)",
               err_name(e.code), e.slot, e.id, h->xl.ghost_cap, h->xl.mig_cap);
      return fail(h, e.code == 6u ? DEM_EOVERFLOW : -(int)e.code, buf);
    }
    h->ids_dense = false;  // ids are global: ORDER_ID is single-GPU only
    // dem_set_contacts maps global ids through a table of id_max + 1 entries
    h->id_bound = hp.id_max < (uint64_t)(4 * n + (1 << 20)) ? (int64_t)hp.id_max + 1 : 0;
    return DEM_OK;
  }
  // 6. ids: unique; dense (a permutation of 0..n-1) enables ORDER_ID and set_contacts
  h->ids_dense = false;
  h->id_bound = 0;
  if (n > 0) {
    uint32_t* seen = nullptr;
    uint32_t* dup = nullptr;
    if (!dalloc(h, &seen, (size_t)n) || !dalloc(h, &dup, 1)) {
      unstage();
      return fail(h, DEM_ENOMEM, "id check allocation failed");
    }
    CUDA_TRY(h, cudaMemsetAsync(seen, 0, sizeof(uint32_t) * n, st));
    CUDA_TRY(h, cudaMemsetAsync(dup, 0, sizeof(uint32_t), st));
    launch_idcheck(st, n, h->ph.idmask, h->omg[0], seen, dup);
    uint32_t hdup = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&hdup, dup, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    dev_free(h, seen);
    dev_free(h, dup);
    if (hp.id_max < (uint64_t)n) {
      if (hdup) {
        unstage();
        h->n = -1;
        return fail(h, DEM_EINVAL, "duplicate particle ids");
      }
      h->ids_dense = true;
      h->id_bound = n;
    } else {
      // sparse ids: check uniqueness on the host (setup path only)
      std::vector<uint32_t> ids((size_t)n);
      std::vector<float4> w((size_t)n);
      CUDA_TRY(h, cudaMemcpyAsync(w.data(), h->omg[0], sizeof(float4) * n,
                                  cudaMemcpyDeviceToHost, st));
      CUDA_TRY(h, cudaStreamSynchronize(st));
      for (int64_t i = 0; i < n; ++i) memcpy(&ids[(size_t)i], &w[(size_t)i].w, 4);
      std::sort(ids.begin(), ids.end());
      if (std::adjacent_find(ids.begin(), ids.end()) != ids.end()) {
        unstage();
        h->n = -1;
        return fail(h, DEM_EINVAL, "duplicate particle ids");
      }
    }
  }
  CUDA_TRY(h, cudaStreamSynchronize(st));
  unstage();
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return DEM_OK;
}

// c̄ above which the dense k_force configuration wins (C2, C3: ~8-11 measured
// faster dense; C4, C5: ~5 faster light; profiles/r1_history.md #25)
constexpr double kDenseContacts = 7.0;

int dem_step(dem_handle* h, int64_t nsteps) {
  if (!h) return DEM_EINVAL;
  if (nsteps < 0) return fail(h, DEM_EINVAL, "nsteps < 0");
  if (h->n < 0) return fail(h, DEM_ESTATE, "dem_step before dem_set_particles");
  if (h->slab && !h->connected) return fail(h, DEM_ESTATE, "slab rank not connected (dem_connect)");
  if (nsteps == 0 || (h->n == 0 && !h->slab)) {
    h->steps += (h->n == 0) ? nsteps : 0;
    return DEM_OK;
  }
  if (h->fcfg < 0) {  // choose the k_force configuration
    const uint32_t fl = h->p.flags;
    if (fl & (DEM_F_FORCE_DENSE | DEM_F_FORCE_LIGHT | DEM_F_FORCE_LANES | DEM_F_FORCE_WS) ||
        h->p.model != DEM_MODEL_PRACTICAL) {
      h->fcfg = (fl & DEM_F_FORCE_WS) ? 3 : (fl & DEM_F_FORCE_LANES) ? 2 : (fl & DEM_F_FORCE_LIGHT) ? 1 : 0;
    } else {
      // one eager step in the dense configuration, then the history entries
      // per particle it produced (c̄, walls included) decide the rest
      h->fcfg = 0;
      h->p.flags |= DEM_F_NO_GRAPH;
      int rc = dem_step(h, 1);
      h->p.flags = fl;
      if (rc) return rc;
      --nsteps;
      if (h->n > 0) {
        dem_stats st{};
        rc = dem_get_stats(h, &st);
        if (rc) return rc;
        const double cbar = (double)st.contacts / (double)h->n;
        h->fcfg = cbar > kDenseContacts ? 0 : 1;
      }
      if (nsteps == 0) return DEM_OK;
    }
  }
  const int64_t ctr0 = h->pending ? h->pend_ctr0 + h->pend_steps : h->steps;
  const int cur0 = h->cur;
  const bool eager = h->profiling || (h->p.flags & DEM_F_NO_GRAPH);
  // merge mode: the first step after dem_set_particles (or a roll-back), and
  // the rest of a call that overflowed the mover capacity, sort by counting
  int64_t nfull = 0;
  if (h->merge && (!h->merge_ok || h->full_run)) nfull = h->full_run ? nsteps : 1;
  if (h->merge) {
    h->merge_ok = true;
    h->full_sorts += nfull;
  }
  if (eager) {
    for (int64_t k = 0; k < nsteps; ++k) {
      int rc = enqueue_step(h, h->cur, h->profiling, k < nfull);
      if (rc) return rc;
      h->cur ^= 1;
    }
    if (h->profiling) {
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      for (auto& pr : h->prof) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.b, pr.e);
        h->kernel_ms[pr.kid] += ms;
        h->kernel_count[pr.kid] += 1;
        h->event_pool.push_back(pr.b);
        h->event_pool.push_back(pr.e);
      }
      h->prof.clear();
    }
  } else {
    auto run = [&](int64_t cnt, bool full) -> int {
      cudaGraphExec_t* G2 = full ? h->gf2 : h->g2;
      cudaGraphExec_t* G1 = full ? h->gf1 : h->g1;
      for (int b = 0; b < 2 && cnt > 0; ++b) {
        if (cnt >= 2 && !G2[b]) {
          int rc = build_graph(h, b, 2, &G2[b], full);
          if (rc) return rc;
        }
        if ((cnt & 1) && !G1[b]) {
          int rc = build_graph(h, b, 1, &G1[b], full);
          if (rc) return rc;
        }
      }
      while (cnt >= 2) {
        CUDA_TRY(h, cudaGraphLaunch(G2[h->cur], h->stream));
        h->graph_launches++;
        h->launches += 2 * kernels_per_step(h, full);
        cnt -= 2;
      }
      if (cnt) {
        CUDA_TRY(h, cudaGraphLaunch(G1[h->cur], h->stream));
        h->graph_launches++;
        h->launches += kernels_per_step(h, full);
        h->cur ^= 1;
      }
      return DEM_OK;
    };
    int rc = run(nfull, true);
    if (rc) return rc;
    rc = run(nsteps - nfull, false);
    if (rc) return rc;
  }
  if (!h->pending) {
    h->pending = true;
    h->pend_ctr0 = ctr0;
    h->pend_cur0 = cur0;
    h->pend_steps = 0;
  }
  h->pend_steps += nsteps;
  h->steps = ctr0 + nsteps;  // provisional until checked
  if (h->p.flags & DEM_F_ASYNC) return DEM_OK;
  return dem_sync(h);
}

int dem_sync(dem_handle* h) {
  if (!h) return DEM_EINVAL;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (!h->pending) return DEM_OK;
  h->pending = false;
  return check_step_error(h, h->pend_ctr0, h->pend_cur0, h->pend_steps);
}

int dem_get_state(dem_handle* h, int32_t order, int64_t cap, const dem_particles* dst,
                  int64_t* n_out) {
  if (!h || !dst) return DEM_EINVAL;
  if (h->pending) {
    int rc = dem_sync(h);
    if (rc) return rc;
  }
  if (h->n < 0) return fail(h, DEM_ESTATE, "no particles set");
  if (n_out) *n_out = h->n;
  if (cap < h->n) return fail(h, DEM_EINVAL, "capacity too small");
  if (order == DEM_ORDER_ID && !h->ids_dense)
    return fail(h, DEM_EINVAL, "DEM_ORDER_ID needs ids 0..n-1");
  if (h->n == 0) return DEM_OK;
  cudaStream_t st = h->stream;
  const int64_t n = h->n;
  const bool dev = dst->mem_kind == DEM_MEM_DEVICE;
  float *o[9] = {dst->pos, dst->vel, dst->omega, dst->radius, dst->mass, (float*)dst->id,
                 dst->force, dst->torque, (float*)dst->material};
  const size_t sz[9] = {3, 3, 3, 1, 1, 1, 3, 3, 1};
  float* d[9] = {};
  std::vector<void*> tmp;
  for (int k = 0; k < 9; ++k) {
    if (!o[k]) continue;
    if (dev) {
      d[k] = o[k];
    } else {
      d[k] = (float*)dev_alloc(h, sizeof(float) * sz[k] * n);
      if (!d[k]) {
        for (void* p : tmp) dev_free(h, p);
        return fail(h, DEM_ENOMEM, "staging allocation failed");
      }
      tmp.push_back(d[k]);
    }
  }
  launch_unpack(st, n, order == DEM_ORDER_ID, h->pos[h->cur], h->vel[h->cur], h->omg[h->cur],
                h->F, h->T, d[0], d[1], d[2], d[3], d[4], (uint32_t*)d[5], d[6], d[7],
                h->ph.idmask, (uint32_t*)d[8]);
  h->launches++;
  if (!dev)
    for (int k = 0; k < 9; ++k)
      if (o[k])
        CUDA_TRY(h, cudaMemcpyAsync(o[k], d[k], sizeof(float) * sz[k] * n,
                                    cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  for (void* p : tmp) dev_free(h, p);
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return DEM_OK;
}

int dem_get_contacts(dem_handle* h, int32_t mem_kind, int64_t cap, uint32_t* id_i,
                     uint32_t* id_j, float* dt3, int64_t* m_out) {
  if (!h) return DEM_EINVAL;
  if (h->pending) {
    int rc = dem_sync(h);
    if (rc) return rc;
  }
  if (h->n < 0) return fail(h, DEM_ESTATE, "no particles set");
  if (h->n == 0 || h->p.model != DEM_MODEL_PRACTICAL) {
    if (m_out) *m_out = 0;
    return DEM_OK;
  }
  cudaStream_t st = h->stream;
  const int64_t n = h->n;
  uint32_t* base = nullptr;
  unsigned long long* status = nullptr;
  uint32_t* ctr = nullptr;
  const uint32_t tiles = (uint32_t)((n + kScanTile - 1) / kScanTile) + 1;
  if (!dalloc(h, &base, (size_t)n + 1) || !dalloc(h, &status, tiles) || !dalloc(h, &ctr, 1))
    return fail(h, DEM_ENOMEM, "allocation failed");
  CUDA_TRY(h, cudaMemsetAsync(status, 0, sizeof(unsigned long long) * tiles, st));
  CUDA_TRY(h, cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
  launch_scan(st, h->cnt[h->cur], base, (uint32_t)n, nullptr, status, ctr, nullptr, 0);
  uint32_t m = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&m, base + n, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  h->launches++;
  if (m_out) *m_out = m;
  int rc = DEM_OK;
  if (cap < (int64_t)m) {
    rc = fail(h, DEM_EINVAL, "capacity too small");
  } else if (m > 0) {
    const bool dev = mem_kind == DEM_MEM_DEVICE;
    uint32_t *di = id_i, *dj = id_j;
    float* dd = dt3;
    if (!dev) {
      di = id_i ? (uint32_t*)dev_alloc(h, 4ull * m) : nullptr;
      dj = id_j ? (uint32_t*)dev_alloc(h, 4ull * m) : nullptr;
      dd = dt3 ? (float*)dev_alloc(h, 12ull * m) : nullptr;
    }
    launch_emit_contacts(st, n, h->cap, h->K, h->hist[h->cur], h->cnt[h->cur], base,
                         h->omg[h->cur], di, dj, dd, h->ph.idmask);
    h->launches++;
    if (!dev) {
      if (id_i) CUDA_TRY(h, cudaMemcpyAsync(id_i, di, 4ull * m, cudaMemcpyDeviceToHost, st));
      if (id_j) CUDA_TRY(h, cudaMemcpyAsync(id_j, dj, 4ull * m, cudaMemcpyDeviceToHost, st));
      if (dt3) CUDA_TRY(h, cudaMemcpyAsync(dt3, dd, 12ull * m, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(h, cudaStreamSynchronize(st));
      dev_free(h, di);
      dev_free(h, dj);
      dev_free(h, dd);
    }
  }
  CUDA_TRY(h, cudaStreamSynchronize(st));
  dev_free(h, base);
  dev_free(h, status);
  dev_free(h, ctr);
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return rc;
}

int dem_set_contacts(dem_handle* h, int32_t mem_kind, int64_t m, const uint32_t* id_i,
                     const uint32_t* id_j, const float* dt3) {
  if (!h || m < 0 || (m > 0 && (!id_i || !id_j || !dt3))) return DEM_EINVAL;
  if (h->n < 0) return fail(h, DEM_ESTATE, "no particles set");
  if (h->id_bound <= 0 && (h->n > 0 || h->slab))
    return fail(h, DEM_EINVAL, h->slab ? "dem_set_contacts needs ids below 4 n + 2^20"
                                       : "dem_set_contacts needs ids 0..n-1");
  if (h->p.model != DEM_MODEL_PRACTICAL) return m == 0 ? DEM_OK : fail(h, DEM_EINVAL, "simple model keeps no history");
  cudaStream_t st = h->stream;
  const int64_t n = h->n;
  CUDA_TRY(h, cudaMemsetAsync(h->cnt[h->cur], 0, sizeof(uint32_t) * (n > 0 ? n : 1), st));
  if (m == 0 || n == 0) {
    CUDA_TRY(h, cudaStreamSynchronize(st));
    return DEM_OK;
  }
  const bool dev = mem_kind == DEM_MEM_DEVICE;
  const uint32_t *di = id_i, *dj = id_j;
  const float* dd = dt3;
  std::vector<void*> tmp;
  if (!dev) {
    void* a = dev_alloc(h, 4ull * m);
    void* b = dev_alloc(h, 4ull * m);
    void* c = dev_alloc(h, 12ull * m);
    tmp = {a, b, c};
    if (!a || !b || !c) {
      for (void* p : tmp) dev_free(h, p);
      return fail(h, DEM_ENOMEM, "allocation failed");
    }
    CUDA_TRY(h, cudaMemcpyAsync(a, id_i, 4ull * m, cudaMemcpyHostToDevice, st));
    CUDA_TRY(h, cudaMemcpyAsync(b, id_j, 4ull * m, cudaMemcpyHostToDevice, st));
    CUDA_TRY(h, cudaMemcpyAsync(c, dt3, 12ull * m, cudaMemcpyHostToDevice, st));
    di = (const uint32_t*)a;
    dj = (const uint32_t*)b;
    dd = (const float*)c;
  } else if (!h->own_stream) {
    cudaStreamSynchronize(nullptr);
  }
  // id -> slot of this handle's particles (slab mode: the owned ones; contacts
  // of particles owned by another rank are skipped)
  uint32_t *slot = nullptr, *flags = nullptr;
  const int64_t nb = h->id_bound;
  if (!dalloc(h, &slot, (size_t)nb) || !dalloc(h, &flags, 1)) {
    for (void* p : tmp) dev_free(h, p);
    return fail(h, DEM_ENOMEM, "allocation failed");
  }
  CUDA_TRY(h, cudaMemsetAsync(flags, 0, 4, st));
  CUDA_TRY(h, cudaMemsetAsync(slot, 0xFF, sizeof(uint32_t) * nb, st));
  launch_slot_of_id(st, n, h->ph.idmask, h->omg[h->cur], slot);
  launch_insert_contacts(st, m, nb, h->cap, h->K, di, dj, dd, slot, h->hist[h->cur], h->cnt[h->cur],
                         flags, h->slab ? 1 : 0);
  h->launches += 2;
  uint32_t hf = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&hf, flags, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  dev_free(h, slot);
  dev_free(h, flags);
  for (void* p : tmp) dev_free(h, p);
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (hf) {
    CUDA_TRY(h, cudaMemset(h->cnt[h->cur], 0, sizeof(uint32_t) * n));
    return fail(h, (hf & 1) ? DEM_EINVAL : DEM_EOVERFLOW,
                (hf & 1) ? "contact id out of range" : "more than max_contacts entries for a particle");
  }
  return DEM_OK;
}

int dem_get_grid(dem_handle* h, int64_t cap, uint32_t* key, uint32_t* perm, uint32_t* off,
                 int64_t* ncells_out) {
  if (!h) return DEM_EINVAL;
  if (h->pending) {
    int rc = dem_sync(h);
    if (rc) return rc;
  }
  if (h->n < 0) return fail(h, DEM_ESTATE, "no particles set");
  if (ncells_out) *ncells_out = h->g.ncells;
  const int64_t n = h->n;
  if ((key || perm) && cap < n) return fail(h, DEM_EINVAL, "capacity too small");
  if (off && cap < (int64_t)h->g.ncells + 1) return fail(h, DEM_EINVAL, "capacity too small");
  cudaStream_t st = h->stream;
  if (key && n) CUDA_TRY(h, cudaMemcpyAsync(key, h->key[h->cur], 4 * n, cudaMemcpyDeviceToHost, st));
  // merge re-sort with one radius: SCCM lives in the sorted positions' .w
  // (k_mv_apply does not write perm on that path)
  if (perm && n && h->merge && step_buffers(h, h->cur).sw_r > 0.f) {
    launch_perm_from_w(st, n, h->pos_sorted, h->perm);
    CUDA_TRY(h, cudaGetLastError());
  }
  if (perm && n) CUDA_TRY(h, cudaMemcpyAsync(perm, h->perm, 4 * n, cudaMemcpyDeviceToHost, st));
  if (off)
    CUDA_TRY(h, cudaMemcpyAsync(off, h->off, 4 * ((size_t)h->g.ncells + 1),
                                cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return DEM_OK;
}

int dem_get_stats(dem_handle* h, dem_stats* out) {
  if (!h || !out) return DEM_EINVAL;
  if (h->pending) {
    int rc = dem_sync(h);
    if (rc) return rc;
  }
  memset(out, 0, sizeof *out);
  out->n = h->n;
  out->ncells = h->g.ncells;
  out->dims[0] = h->g.nx;
  out->dims[1] = h->g.ny;
  out->dims[2] = h->g.nz;
  out->cell_edge = h->h;
  out->steps = h->steps;
  out->launches = h->launches;
  out->graph_launches = h->graph_launches;
  out->force_cfg = h->fcfg;
  out->fused_sweep = fused_sweep(h) ? 1 : 0;
  out->full_sorts = (int32_t)h->full_sorts;
  for (int k = 0; k < 8; ++k) {
    out->kernel_ms[k] = h->kernel_ms[k];
    out->kernel_count[k] = h->kernel_count[k];
  }
  if (h->n > 0) {
    uint32_t* ms = nullptr;
    if (!dalloc(h, &ms, 1)) return fail(h, DEM_ENOMEM, "allocation failed");
    CUDA_TRY(h, cudaMemsetAsync(ms, 0, 4, h->stream));
    launch_max_speed(h->stream, h->n, h->vel[h->cur], ms);
    uint32_t hb = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&hb, ms, 4, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    dev_free(h, ms);
    float f;
    memcpy(&f, &hb, 4);
    out->max_speed = f;
  }
  if (h->n > 0 && h->p.model == DEM_MODEL_PRACTICAL) {
    unsigned long long* sm = nullptr;
    if (!dalloc(h, &sm, 2)) return fail(h, DEM_ENOMEM, "allocation failed");
    CUDA_TRY(h, cudaMemsetAsync(sm, 0, 16, h->stream));
    launch_cnt_stats(h->stream, h->n, h->cnt[h->cur], sm);
    unsigned long long hs[2] = {0, 0};
    CUDA_TRY(h, cudaMemcpyAsync(hs, sm, 16, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    dev_free(h, sm);
    out->contacts = (int64_t)hs[0];
    out->max_contacts_seen = (int64_t)hs[1];
  }
  return DEM_OK;
}

int dem_analyze(dem_handle* h, dem_analysis* out) {
  if (!h || !out) return DEM_EINVAL;
  if (h->n < 0 || h->steps == 0) return fail(h, DEM_ESTATE, "dem_analyze before the first step");
  int rc = dem_sync(h);
  if (rc) return rc;
  std::memset(out, 0, sizeof(*out));
  unsigned long long* acc = nullptr;
  constexpr int kAcc = 9 + 33;
  if (!dalloc(h, &acc, kAcc)) return fail(h, DEM_ENOMEM, "allocation failed");
  CUDA_TRY(h, cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * kAcc, h->stream));
  // the last step read parity cur ^ 1; its sort, offsets and contact lists are intact
  launch_analyze(h->stream, h->cap, step_buffers(h, h->cur ^ 1), h->g, acc);
  unsigned long long a[kAcc];
  CUDA_TRY(h, cudaMemcpyAsync(a, acc, sizeof(a), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  dev_free(h, acc);
  out->n = (int64_t)a[0];
  out->candidates = (int64_t)a[1];
  out->max_candidates = (int64_t)a[2];
  out->contacts = (int64_t)a[3];
  out->max_contacts = (int64_t)a[4];
  out->warp_candidate_slots = (int64_t)a[5];
  out->warp_contact_slots = (int64_t)a[6];
  out->max_per_cell = (int64_t)a[7];
  out->occupied_cells = (int64_t)a[8];
  for (int k = 0; k < 33; ++k) out->contact_hist[k] = (int64_t)a[9 + k];
  out->movers = -1;
  if (h->merge) {
    uint32_t m = 0;  // the movers the next step will merge (listed by the last step)
    CUDA_TRY(h, cudaMemcpy(&m, h->mov_n + h->cur, sizeof m, cudaMemcpyDeviceToHost));
    out->movers = (int64_t)m;
  }
  return DEM_OK;
}

int dem_profile(dem_handle* h, int32_t enable) {
  if (!h) return DEM_EINVAL;
  h->profiling = enable != 0;
  if (h->profiling) {
    for (int k = 0; k < 8; ++k) {
      h->kernel_ms[k] = 0.0;
      h->kernel_count[k] = 0;
    }
  }
  return DEM_OK;
}

int dem_exchange_handle(dem_handle* h, void* out64) {
  if (!h || !out64) return DEM_EINVAL;
  if (!h->slab || !h->xregion) return fail(h, DEM_ESTATE, "no exchange region (set particles first)");
  cudaIpcMemHandle_t m;
  CUDA_TRY(h, cudaIpcGetMemHandle(&m, h->xregion));
  memcpy(out64, &m, sizeof m);
  return DEM_OK;
}

int dem_exchange_ptr(dem_handle* h, void** out) {
  if (!h || !out) return DEM_EINVAL;
  if (!h->slab || !h->xregion) return fail(h, DEM_ESTATE, "no exchange region (set particles first)");
  *out = h->xregion;
  return DEM_OK;
}

// Both neighbours must have published the same exchange layout as this rank
// (their blocks are read at this rank's offsets): the same particle set was
// given to every rank.
static int check_peer_layouts(dem_handle* h) {
  const uint8_t* peers[2] = {h->xleft, h->xright};
  for (const uint8_t* p : peers) {
    if (!p) continue;
    XLayout pl{};
    CUDA_TRY(h, cudaMemcpy(&pl, p, sizeof pl, cudaMemcpyDeviceToHost));
    if (pl.bytes != h->xl.bytes || pl.mig_cap != h->xl.mig_cap ||
        pl.ghost_cap != h->xl.ghost_cap || pl.K != h->xl.K || pl.mono_bits != h->xl.mono_bits ||
        pl.plane != h->xl.plane)
      return fail(h, DEM_EINVAL,
                  "neighbour exchange layout differs (ghost capacity " + std::to_string(pl.ghost_cap) +
                      " vs " + std::to_string(h->xl.ghost_cap) +
                      "): give every rank the same particle set in dem_set_particles");
  }
  return DEM_OK;
}

int dem_connect(dem_handle* h, const void* left64, const void* right64) {
  if (!h) return DEM_EINVAL;
  if (!h->slab) return fail(h, DEM_ESTATE, "not a slab rank");
  const void* in[2] = {left64, right64};
  const uint8_t** outp[2] = {&h->xleft, &h->xright};
  bool* ipc[2] = {&h->xleft_ipc, &h->xright_ipc};
  for (int k = 0; k < 2; ++k) {
    if (!in[k]) {
      *outp[k] = nullptr;
      continue;
    }
    cudaIpcMemHandle_t m;
    memcpy(&m, in[k], sizeof m);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, m, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(h, DEM_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    *outp[k] = (const uint8_t*)p;
    *ipc[k] = true;
  }
  if ((h->rank > 0) != (h->xleft != nullptr) || (h->rank < h->world - 1) != (h->xright != nullptr))
    return fail(h, DEM_EINVAL, "a rank needs exactly its existing neighbours");
  int rc = check_peer_layouts(h);
  if (rc) return rc;
  h->connected = true;
  destroy_graphs(h);
  return DEM_OK;
}

int dem_connect_ptrs(dem_handle* h, void* left, void* right) {
  if (!h) return DEM_EINVAL;
  if (!h->slab) return fail(h, DEM_ESTATE, "not a slab rank");
  h->xleft = (const uint8_t*)left;
  h->xright = (const uint8_t*)right;
  h->xleft_ipc = h->xright_ipc = false;
  if ((h->rank > 0) != (h->xleft != nullptr) || (h->rank < h->world - 1) != (h->xright != nullptr))
    return fail(h, DEM_EINVAL, "a rank needs exactly its existing neighbours");
  int rc = check_peer_layouts(h);
  if (rc) return rc;
  h->connected = true;
  destroy_graphs(h);
  return DEM_OK;
}

}  // extern "C"

// dem_kernels.cu — the sm_100a kernels of one DEM timestep (arXiv 1301.1714).
//
// One step on the default single-GPU path (§4.2):
// k_merge and k_force with the detection inside it (one radius), or k_merge,
// k_detect, k_force (per-particle radii, DEM_F_SPLIT_SWEEP):
//   k_merge   steps 3-4: the stable sort of Eq. 11 as a merge of the few
//             particles that changed cell into the last sorted order (every
//             quantity is a count over the mover list the integrator made);
//             SCCM travels in the sorted positions, the cell offsets (SPEC
//             cell ranges) are shifted in place.
//   k_detect  steps 5-6: one thread per sorted slot scans the 27 cells of
//             Eq. 12 with the fp64-defined contact predicate (R14) and writes
//             its contact list and its warp-flattened (base, count) word.
//             (One radius: the same scan runs inside k_force<..., FUSED>,
//             its lists in shared memory, each z-plane's rows as one run.)
//   k_force   steps 7-8, 1 and the next step's 2: a warp per 32 sorted slots
//             deals its contacts 32 per round to all lanes (Eqs. 2-10 with the
//             tangential history remapped through the old slots, Eq. 7), then
//             each particle adds its contacts in candidate order, applies the
//             walls, integrates, writes its state at the sorted slot (step 4's
//             reorder), hashes the new position and lists itself if it changed
//             cell.
// The first step after dem_set_particles (and a step whose movers overflow
// the list) sorts by counting instead: k_count/k_tile_sum/k_scan_apply (the
// scan is the offset array), k_scatter, k_rank. Slab ranks add the exchange
// kernels (k_xrecv at the step start, k_xghost_place after the sort,
// k_xpack_planes + k_xpack_write at the end).
// All arithmetic of the step runs here; the host only enqueues.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "dem_internal.h"

#ifndef DEM_ABLATIONS  // 1: also build the ablation kernels (libdem_ablations.so)
#define DEM_ABLATIONS 0
#endif

namespace dem {

// ------------------------------------------------------------ helpers ------

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch (launch_pdl): let the next kernel of the step
// be scheduled while this one drains, then wait here until the previous
// kernel has completed and its writes are visible. No-ops when launched
// without the attribute.
#ifndef DEM_PDL
#define DEM_PDL 0  // measured: no gain in the graph (profiles/r1_history.md #24)
#endif
__device__ __forceinline__ void pdl_enter() {
#if DEM_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Record the first error of a step (positive code); later errors are ignored.
__device__ void raise_error(DevErr* e, uint32_t code, uint32_t slot, uint32_t id) {
  if (atomicCAS(&e->code, 0u, code) == 0u) {
    e->slot = slot;
    e->id = id;
    e->step = ld_volatile(&e->step_ctr);
    __threadfence();
  }
}

// Step 2: the cell of a position, as the fp64 expression of
// R15: c_a = clamp(floor((x_a - lo_a) * inv_h), 0, n_a - 1). __dsub_rn and
// __dmul_rn keep it two correctly rounded operations.
__device__ __forceinline__ int cell_coord(float x, double lo, double inv_h, int n) {
  // floor and int conversion in one cvt.rmi (saturating; NaN -> 0), then the
  // clamp in integers: the same cell as flooring and clamping in fp64
  const int c = __double2int_rd(__dmul_rn(__dsub_rn((double)x, lo), inv_h));
  return min(max(c, 0), n - 1);
}

// Local cell key of a position: global (cx, cy, cz) of R15, z shifted to the
// rank's local planes. Returns the trash key for a z outside the local grid
// (only reachable in slab mode; the caller flags it).
__device__ __forceinline__ uint32_t cell_key(const DevGrid& g, float x, float y, float z) {
  int cx = cell_coord(x, g.lo[0], g.inv_h, g.nx);
  int cy = cell_coord(y, g.lo[1], g.inv_h, g.ny);
  int cz = cell_coord(z, g.lo[2], g.inv_h, g.nz_global) - g.zlo;
  if (cz < 0 || cz >= g.nz) return g.trash;
  return (uint32_t)cx + (uint32_t)g.nx * ((uint32_t)cy + (uint32_t)g.ny * (uint32_t)cz);
}

// Counting-sort contribution of one particle: warp-aggregated atomic on its
// cell (lanes with the same key share one atomic; __match_any_sync groups
// them), returning its (arbitrary but unique) rank inside the cell.
__device__ __forceinline__ uint32_t count_into_cell(uint32_t* count, uint32_t key) {
  const uint32_t active = __activemask();
  const uint32_t peers = __match_any_sync(active, key);
  const uint32_t leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (lane_id() == leader) base = atomicAdd(&count[key], (uint32_t)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + (uint32_t)__popc(peers & lanemask_lt());
}

struct f3 {
  float x, y, z;
};
__device__ __forceinline__ f3 mk(float x, float y, float z) { return {x, y, z}; }
__device__ __forceinline__ float dot(f3 a, f3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ f3 cross(f3 a, f3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Tangential history (Eq. 7 δ_t) layout: slot-major, entry k of slot j at
// j K + k, so the contacts of one particle — consecutive lanes of a k_force
// round — read and write one contiguous run.
__device__ __forceinline__ size_t hix(uint32_t slot, uint32_t k, uint32_t K) {
  return (size_t)slot * K + k;
}

// Approximate MUFU reciprocal / square root (|rel. error| ~ 2^-22): the
// force arithmetic is fp32 with a 1e-4 parity tolerance, and IEEE div/sqrt
// expand into slow-path subroutines. Deterministic, so the pair evaluation
// stays bitwise antisymmetric (P11).
__device__ __forceinline__ float frcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fsqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------ set_particles kernels ----

__global__ void k_probe(int64_t n, PackIn in, DevGrid g, Probe* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float r = in.radius ? in.radius[i] : in.def_radius;
  float m = in.mass ? in.mass[i] : in.def_mass_coef * r * r * r;
  if (!(r > 0.0f) || !isfinite(r)) atomicAdd(&out->bad_radius, 1u);
  if (!(m > 0.0f) || !isfinite(m)) atomicAdd(&out->bad_mass, 1u);
  bool fin = true;
  for (int a = 0; a < 3; ++a) {
    float x = in.pos[3 * i + a];
    fin &= isfinite(x);
    if (in.vel) fin &= isfinite(in.vel[3 * i + a]);
    if (in.omega) fin &= isfinite(in.omega[3 * i + a]);
    // a centre may lie up to r beyond a wall (in contact with it): the states
    // a step produces (R18) must be loadable again
    if (isfinite(x) && ((double)x < g.lo[a] - (double)r || (double)x > g.hi[a] + (double)r))
      atomicAdd(&out->outside, 1u);
  }
  if (!fin) atomicAdd(&out->nonfinite, 1u);
  if (r > 0.0f && isfinite(r)) {
    atomicMax(&out->rmax_bits, __float_as_uint(r));
    atomicMax(&out->rmin_cbits, ~__float_as_uint(r));
  }
  uint32_t id = in.id ? in.id[i] : (uint32_t)i;
  if (id >= kWallPid0 || (in.nmat > 1 && id >= (1u << kMatShift))) atomicAdd(&out->bad_id, 1u);
  if (in.nmat > 1 && in.material && in.material[i] >= in.nmat) atomicAdd(&out->bad_material, 1u);
  atomicMax(&out->id_max, id);
}

__global__ void k_pack(int64_t n, PackIn in, DevGrid g, float4* pos, float4* vel, float4* omg,
                       uint32_t* key, uint32_t* count, uint32_t* prank, const uint32_t* dst,
                       const uint32_t* keep) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t src = i;
  if (keep) {  // slab mode: only this rank's particles, compacted in input order
    if (!keep[i]) return;
    i = dst[i];
  }
  const int64_t q = src;
  float r = in.radius ? in.radius[q] : in.def_radius;
  float m = in.mass ? in.mass[q] : in.def_mass_coef * r * r * r;
  float x = in.pos[3 * q], y = in.pos[3 * q + 1], z = in.pos[3 * q + 2];
  pos[i] = make_float4(x, y, z, r);
  vel[i] = in.vel ? make_float4(in.vel[3 * q], in.vel[3 * q + 1], in.vel[3 * q + 2], m)
                  : make_float4(0.f, 0.f, 0.f, m);
  uint32_t id = in.id ? in.id[q] : (uint32_t)q;
  if (in.nmat > 1 && in.material) id |= in.material[q] << kMatShift;  // the id word
  omg[i] = in.omega
               ? make_float4(in.omega[3 * q], in.omega[3 * q + 1], in.omega[3 * q + 2],
                             __uint_as_float(id))
               : make_float4(0.f, 0.f, 0.f, __uint_as_float(id));
  uint32_t k = cell_key(g, x, y, z);
  key[i] = k;
  prank[i] = count_into_cell(count, k);
}

__global__ void k_count(int64_t n, const uint32_t* key, uint32_t* count, uint32_t* prank) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  prank[i] = count_into_cell(count, key[i]);
}

// Duplicate-id check for dense ids (max id < n): seen[] is zeroed by the host.
__global__ void k_idcheck(int64_t n, uint32_t idmask, const float4* omg, uint32_t* seen,
                          uint32_t* dup) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t id = __float_as_uint(omg[i].w) & idmask;
  if (id < (uint64_t)n && atomicExch(&seen[id], 1u) != 0u) atomicAdd(dup, 1u);
}

// ------------------------------------------------------------ k_scan -------
// Exclusive scan out[0..n] of in[0..n) (out[n] = total) in two passes of
// 4,096-element tiles: k_tile_sum writes one sum per tile; k_scan_apply adds
// the sums of all preceding tiles (a block-wide reduction over at most a few
// thousand L2-resident words) to the tile's own block scan. No inter-block
// waiting, so every tile streams at full bandwidth. Optionally zeroes `zero`
// (the per-cell counts, ready for the next step's atomics) and advances the
// step counter. `in` and `zero` may alias.

__device__ __forceinline__ void load_tile(const uint32_t* in, uint32_t n, uint64_t base,
                                          uint32_t (&v)[kScanItems]) {
  if (base + kScanItems <= n) {
    const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const uint4 w = __ldcs(&p[q]);
      v[4 * q] = w.x;
      v[4 * q + 1] = w.y;
      v[4 * q + 2] = w.z;
      v[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) v[q] = (base + q < n) ? in[base + q] : 0u;
  }
}

__device__ __forceinline__ uint32_t block_sum(uint32_t x, uint32_t* s_warp) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
  __syncthreads();
  if (lane == 0) s_warp[warp] = x;
  __syncthreads();
  uint32_t t = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
  return t;
}

__global__ void __launch_bounds__(kScanThreads)
    k_tile_sum(const uint32_t* in, uint32_t n, uint32_t* tsum, DevErr* err, int count_step) {
  pdl_enter();
  __shared__ uint32_t s_warp[kScanThreads / 32];
  const uint32_t e = err ? ld_volatile(&err->code) : 0u;  // checked once the loads are out
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  load_tile(in, n, base, v);
  if (e != 0u) return;
  uint32_t local = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) local += v[q];
  const uint32_t tot = block_sum(local, s_warp);
  if (threadIdx.x == 0) {
    tsum[blockIdx.x] = tot;
    if (blockIdx.x == 0 && count_step && err) atomicAdd(&err->step_ctr, 1u);
  }
}

__global__ void __launch_bounds__(kScanThreads)
    k_scan_apply(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* zero,
                 const uint32_t* __restrict__ tsum, DevErr* err, uint32_t base0) {
  pdl_enter();
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_excl[kScanThreads / 32];
  const uint32_t e = err ? ld_volatile(&err->code) : 0u;  // checked once the loads are out
  const uint32_t tile = blockIdx.x;
  const uint64_t base = (uint64_t)tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  load_tile(in, n, base, v);
  // prefix of all preceding tiles
  uint32_t acc = 0;
  for (uint32_t t = threadIdx.x; t < tile; t += kScanThreads) acc += __ldg(&tsum[t]);
  if (e != 0u) return;
  const uint32_t prefix = base0 + block_sum(acc, s_warp);
  uint32_t local = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) local += v[q];
  // block exclusive scan of `local`
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t incl = local;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= (uint32_t)d) incl += t;
  }
  __syncthreads();
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int d = 1; d < kScanThreads / 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= (uint32_t)d) wi += t;
    }
    if (lane < kScanThreads / 32) s_excl[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1 && (uint64_t)(tile + 1) * kScanTile >= n)
      out[n] = prefix + wi;  // total
  }
  __syncthreads();
  uint32_t run = prefix + s_excl[warp] + (incl - local);
  if (base + kScanItems <= n) {
    uint4* p = reinterpret_cast<uint4*>(out + base);
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      uint4 w;
      w.x = run;
      run += v[4 * q];
      w.y = run;
      run += v[4 * q + 1];
      w.z = run;
      run += v[4 * q + 2];
      w.w = run;
      run += v[4 * q + 3];
      p[q] = w;
    }
    if (zero) {
      uint4* z = reinterpret_cast<uint4*>(zero + base);
#pragma unroll
      for (int q = 0; q < kScanItems / 4; ++q) __stcs(&z[q], make_uint4(0u, 0u, 0u, 0u));
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanItems; ++q)
      if (base + q < n) {
        out[base + q] = run;
        run += v[q];
        if (zero) zero[base + q] = 0u;
      }
  }
}

// --------------------------------------------------------- k_scatter -------
// Four slots per thread, loads batched ahead of the dependent off[] gathers so
// every thread keeps several independent memory requests in flight.
constexpr int kItems = 4;

__global__ void __launch_bounds__(256)
    k_scatter(int64_t n, const uint32_t* __restrict__ nslots, const uint32_t* __restrict__ key,
              const uint32_t* __restrict__ prank, const uint32_t* __restrict__ off,
              uint32_t* __restrict__ tmp, const DevErr* err) {
  pdl_enter();
  // error word, slot count and the first loads go out together (loads below
  // the capacity n are always in bounds; entries past nslots are ignored)
  const uint32_t e = ld_volatile(&err->code);
  const int64_t ns = (int64_t)__ldg(nslots);  // this step's input slots
  const int64_t base = (int64_t)blockIdx.x * blockDim.x * kItems + threadIdx.x;
  uint32_t k[kItems], r[kItems], o[kItems];
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const int64_t i = base + (int64_t)u * blockDim.x;
    k[u] = i < n ? __ldg(&key[i]) : 0u;
    r[u] = i < n ? __ldg(&prank[i]) : 0u;
  }
  if (e != 0u) return;
  n = min(n, ns);
#pragma unroll
  for (int u = 0; u < kItems; ++u) o[u] = base + (int64_t)u * blockDim.x < n ? __ldg(&off[k[u]]) : 0u;
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const int64_t i = base + (int64_t)u * blockDim.x;
    if (i < n) tmp[o[u] + r[u]] = (uint32_t)i;
  }
}

// ------------------------------------------------------------ k_rank -------
// perm[off[c] + #{t in cell c: tmp[t] < s}] = s, and the particle's position
// gathered into sorted order (PAPER.md:125 step 4, for the field the 27-cell
// candidate loop reads; velocities and spins are read through SCCM).
__global__ void __launch_bounds__(256)
    k_rank(int64_t n, const uint32_t* __restrict__ key, const uint32_t* __restrict__ off,
           const uint32_t* __restrict__ tmp, uint32_t* __restrict__ perm,
           const float4* __restrict__ pos_in, float4* __restrict__ pos_sorted,
           const uint32_t* __restrict__ nslots, const DevErr* err, bool sw, uint32_t base0) {
  pdl_enter();
  // error word, slot count and the first loads go out together (tmp below the
  // capacity n is always in bounds; entries past nslots are ignored). The
  // sorted slots start at base0 (slab ranks: past the left ghost plane's room)
  const uint32_t ecode = ld_volatile(&err->code);
  const int64_t ns = (int64_t)__ldg(nslots);
  const int64_t base = (int64_t)blockIdx.x * blockDim.x * kItems + threadIdx.x;
  uint32_t s[kItems], c[kItems], a[kItems], e[kItems];
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const int64_t j = base0 + base + (int64_t)u * blockDim.x;
    s[u] = j < n ? __ldg(&tmp[j]) : 0u;
  }
  if (ecode != 0u) return;
  n = min(n, ns);
#pragma unroll
  for (int u = 0; u < kItems; ++u) c[u] = base + (int64_t)u * blockDim.x < n ? __ldg(&key[s[u]]) : 0u;
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const bool ok = base + (int64_t)u * blockDim.x < n;
    a[u] = ok ? __ldg(&off[c[u]]) : 0u;
    e[u] = ok ? __ldg(&off[c[u] + 1]) : 0u;
  }
  float4 P[kItems];
#pragma unroll
  for (int u = 0; u < kItems; ++u)
    P[u] = base + (int64_t)u * blockDim.x < n ? __ldcs(&pos_in[s[u]]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    if (base + (int64_t)u * blockDim.x >= n) continue;
    uint32_t r = 0;
    for (uint32_t t = a[u]; t < e[u]; ++t) r += (__ldg(&tmp[t]) < s[u]) ? 1u : 0u;
    perm[a[u] + r] = s[u];
    if (sw) P[u].w = __uint_as_float(s[u]);  // one radius: .w carries the old slot
    pos_sorted[a[u] + r] = P[u];
  }
}

// ------------------------------------------- merge re-sort -----
// Between two steps a particle rarely changes cell (|Δx| per step << h), and
// the state is stored in the previous step's sorted order. So the stable sort
// of Eq. 11 (ties by current slot, R16) is a merge: the *stayers* (slots whose
// new key equals the previous SCM there) are already in order; only the few
// *movers* need placing. With A = the mover slots a_i, their new keys c_i,
// previous keys c'_i and insertion points x_i = clamp(a_i, off[c_i],
// off[c_i+1]) among the stayers (previous offsets: a stayer at slot s
// precedes mover i exactly when s < x_i, because the previous SCM is
// non-decreasing in the slot), the stable order is
//   stayer s -> s + #{i: x_i <= s} - #{i: a_i <= s},
//   mover i  -> r_i + x_i - #{j: a_j < x_i},  r_i = #{j: (c_j, a_j) < (c_i, a_i)},
//   off'[c]   = off[c] + #{i: c_i < c} - #{i: c'_i < c}.
// Every one of these is a count over the mover list, so one kernel places
// everything with no sort at all: block b takes the slots and the cells
// [1024 b, 1024 b + 1024), counts the movers below its range (a block
// reduction over the list, which stays in L2), collects the few events
// inside it in shared memory, and moves its stayers and shifts its offsets;
// block b also places movers b, b + grid, ... (a block-wide count each).
// Bit-identical to the counting sort (the same unique stable permutation).
// The integrator of the previous step listed the movers as (a, c, c', x)
// (finish_particle: it has the sorted slot, both keys and these offsets);
// more than the capacity raises code 12 and the host redoes that step with
// the counting sort. (Round 1 sorted the movers in one block first and built
// per-block event tables: 20-30 us on one SM per step on C4.)
#ifndef DEM_MERGE_SPAN
#define DEM_MERGE_SPAN 1024
#endif
constexpr uint32_t kMergeSpan = DEM_MERGE_SPAN;  // slots and cells per k_merge block
constexpr int kMergeItems = kMergeSpan / 256;
constexpr uint32_t kMergeEv = 512;     // in-block events held in shared memory

// two block sums (256 threads) with one pair of barriers
__device__ __forceinline__ int2 block_sum2(int a, int c, int2* red) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, d);
    c += __shfl_xor_sync(0xffffffffu, c, d);
  }
  __syncthreads();  // (red reused)
  if ((threadIdx.x & 31u) == 0u) red[threadIdx.x >> 5] = make_int2(a, c);
  __syncthreads();
  int2 s = make_int2(0, 0);
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    s.x += red[w].x;
    s.y += red[w].y;
  }
  return s;
}
__device__ __forceinline__ int block_sum(int v, int* red) {  // 256 threads
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  __syncthreads();  // (red reused)
  if ((threadIdx.x & 31u) == 0u) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int s = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w];
  return s;
}

constexpr uint32_t kXDep = 1024;  // departed particles per ghost plane held in shared memory

// After the owned sort: the neighbours' boundary planes (already sorted by
// their keys, with their cell offsets) become this rank's ghost planes,
// merged with this rank's own departed particles of that plane (listed by
// the last integrator with insertion point 0xFFFFFFFF): within a cell the
// departed ones come first, in slot order — the stable order of a sort over
// this rank's input slots, where departed particles (outputs) precede the
// appended planes. Left plane right-aligned below gl_base, right plane
// right after the owned particles; the ghost cells' offsets, then the trash
// cell's and the total. One thread per ghost cell.
struct GhostSmem {
  uint2 dep[kXDep];  // (key, slot) of this side's departed particles
  uint32_t nd, ins, rem;
};

// One block `pb` of the 2 x half ghost-placement blocks. end_from_list: the
// owned particles' end (the right plane's start) counted from the mover list
// (gl_base + n + insertions - removals), for blocks that run beside the
// merge that places the owned particles; else read from off[own_c1].
__device__ __forceinline__ void ghost_place_block(const StepBuffers& b, const DevGrid& g, uint32_t N,
                                                  const uint8_t* left, const uint8_t* right,
                                                  const XLayout& L, XState* xs, uint32_t par,
                                                  uint32_t pb, uint32_t half, bool end_from_list,
                                                  uint32_t n_own_in, GhostSmem& sm) {
  const uint32_t P = L.plane;
  const int side = pb < half ? 0 : 1;  // 0: the left ghost plane
  const uint32_t k = (pb - (side ? half : 0)) * blockDim.x + threadIdx.x;  // plane cell
  const uint8_t* peer = side == 0 ? left : right;
  const uint32_t cf = side == 0 ? 0u : g.own_c1;  // the ghost plane's first cell
  // this side's departed particles from the mover list (and its counts)
  if (threadIdx.x == 0) sm.nd = sm.ins = sm.rem = 0u;
  __syncthreads();
  const uint32_t m = min(ld_volatile(b.mv.n_in), b.mv.cap);
  uint32_t ins = 0, rem = 0;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint4 v = __ldcg(&b.mv.list_in[i]);
    if (peer && v.w == 0xFFFFFFFFu && v.y - cf < P) {
      const uint32_t d = atomicAdd(&sm.nd, 1u);
      if (d < kXDep) sm.dep[d] = make_uint2(v.y, v.x);
    }
    ins += v.w != 0xFFFFFFFFu ? 1u : 0u;
    rem += v.x < n_own_in ? 1u : 0u;
  }
  if (end_from_list) {
    atomicAdd(&sm.ins, ins);
    atomicAdd(&sm.rem, rem);
  }
  __syncthreads();
  const uint32_t end_own = end_from_list ? b.gl_base + n_own_in + sm.ins - sm.rem
                                         : __ldg(&b.off[g.own_c1]);
  if (!peer) {  // no neighbour on this side: no ghost plane (the trash cell and the total)
    if (side == 1 && k == 0) {
      b.off[g.trash] = end_own;
      b.off[g.ncells] = end_own;
    }
    return;
  }
  const uint32_t nd = sm.nd;
  if (nd > kXDep) {
    if (k == 0) raise_error(b.err, 6u, cf, nd);
    return;
  }
  const uint32_t nG = xs->appended[2 + side];
  const uint32_t gs = xs->n_out + xs->appended[0] + xs->appended[1] + (side ? xs->appended[2] : 0u);
  const uint32_t base = side == 0 ? b.gl_base - nG - nd : end_own;
  if ((side == 0 && nG + nd > b.gl_base) || (uint64_t)base + nG + nd > N) {
    if (k == 0) raise_error(b.err, 6u, cf, nG + nd);
    return;
  }
  if (k > P) return;
  const uint8_t* blk = peer + (size_t)((side == 0 ? 1 : 0) * 2 + par) * L.bytes;
  const uint32_t* goff = reinterpret_cast<const uint32_t*>(blk + L.gh_off);
  const uint32_t c = cf + k;
  uint32_t d_lt = 0, d_eq = 0;  // departed particles in cells below c, in c
  for (uint32_t d = 0; d < nd; ++d) {
    d_lt += sm.dep[d].x < c ? 1u : 0u;
    d_eq += sm.dep[d].x == c ? 1u : 0u;
  }
  const uint32_t g0 = __ldcv(goff + k);
  const uint32_t start = base + g0 + d_lt;  // the cell's first sorted slot
  const bool sw = b.sw_r > 0.f;
  auto place = [&](uint32_t j, uint32_t q) {  // sorted slot j <- input slot q
    float4 S = __ldg(&b.pos_in[q]);
    if (sw) S.w = __uint_as_float(q);
    else b.perm[j] = q;
    b.pos_sorted[j] = S;
  };
  if (k == P) {  // one past the plane: the owned particles' start / the trash cell
    if (side == 1) {
      b.off[g.trash] = start;
      b.off[g.ncells] = start;
    }
    return;
  }
  b.off[c] = start;
  // within a cell, where one sorted order of all the particles (a single
  // GPU's) puts them: this rank's departed particles came from the plane
  // above the left ghost plane (later slots: after the cell's particles)
  // and from the plane below the right one (earlier slots: before them)
  const uint32_t g1 = __ldcv(goff + k + 1);
  const uint32_t dep0 = side == 0 ? start + (g1 - g0) : start;  // the departed ones' first slot
  const uint32_t gh0 = side == 0 ? start : start + d_eq;        // the received ones' first slot
  if (d_eq) {  // departed particles of this cell, in slot order
    for (uint32_t d = 0; d < nd; ++d) {
      if (sm.dep[d].x != c) continue;
      uint32_t r = 0;
      for (uint32_t e = 0; e < nd; ++e)
        r += (sm.dep[e].x == c && sm.dep[e].y < sm.dep[d].y) ? 1u : 0u;
      place(dep0 + r, sm.dep[d].y);
    }
  }
  for (uint32_t i = g0; i < g1; ++i) place(gh0 + (i - g0), gs + i);
}

// Slab ranks: n from n_dev (the previous step's owned outputs), sorted slots
// from `base` (constant across steps), offsets of cells [c_lo, c_hi] only; a
// list entry with insertion point 0xFFFFFFFF (a migrant that left) is a
// removal only, one with previous key 0xFFFFFFFF (an arrived migrant,
// appended past the outputs) an insertion only. Single GPU: n_dev null,
// base 0, [0, ncells].
struct GhostArgs {  // slab ranks: the ghost-placement blocks that run beside the merge
  StepBuffers b;
  DevGrid g;
  const uint8_t *left, *right;
  XLayout L;
  XState* xs;
  uint32_t N;
  uint32_t nghost;  // blocks at the end of k_merge's grid (0: single GPU)
};

// GH: slab ranks, the ghost planes placed by the last ga.nghost blocks
template <bool GH>
__global__ void __launch_bounds__(256)
    k_merge(uint32_t n, uint32_t ncells, MergeBuffers mb, const float4* __restrict__ pos_in,
            uint32_t* __restrict__ perm, float4* __restrict__ pos_sorted,
            uint32_t* __restrict__ off, DevErr* err, bool sw, const uint32_t* n_dev,
            uint32_t base, uint32_t c_lo, uint32_t c_hi, const __grid_constant__ GhostArgs ga) {
  pdl_enter();
  __shared__ int red[2][8];
  __shared__ int2 red2[8];
  __shared__ uint32_t s_ne[2];
  __shared__ int2 s_ev[2][kMergeEv];  // (position, weight): slot events, cell events
  const uint32_t b = blockIdx.x, t = threadIdx.x;
  const uint32_t B0 = b * kMergeSpan;
  // the error word, the mover count and this block's positions go out together
  const uint32_t e = ld_volatile(&err->code);
  const uint32_t m = ld_volatile(mb.n_in);
  if (GH) n = *n_dev;
  if (!GH) {  // (single GPU: every slot and cell from 0)
    base = 0u;
    c_lo = 0u;
    c_hi = ncells;
  }
  const uint32_t mgrid = GH ? gridDim.x - ga.nghost : gridDim.x;  // the merge's own blocks
  if (GH && b >= mgrid) {  // slab: place the ghost planes (they need no result of the merge)
    __shared__ GhostSmem gsm;
    if (e != 0u || m > mb.cap) return;
    ghost_place_block(ga.b, ga.g, ga.N, ga.left, ga.right, ga.L, ga.xs, ga.xs->pad[0] & 1u,
                      b - mgrid, ga.nghost / 2, true, n, gsm);
    return;
  }
  float4 P[kMergeItems];
#pragma unroll
  for (int u = 0; u < kMergeItems; ++u) {
    const uint32_t s = B0 + u * 256u + t;
    P[u] = s < n ? __ldcs(&pos_in[s]) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (e != 0u) return;
  if (b == 0 && t == 0) {
    atomicAdd(&err->step_ctr, 1u);  // (the counting sort's k_tile_sum does it otherwise)
    if (m > mb.cap) raise_error(err, 12u, m, 0u);  // (recorded as this step)
    else *mb.n_out = 0u;  // this step's integrator lists the next movers
  }
  if (m > mb.cap) return;  // more movers than listed: the host redoes the step by counting
  if (t < 2) s_ne[t] = 0u;
  __syncthreads();
  // movers below this block's slots / cells, and the events inside them
  int dS = 0, dC = 0;
  for (uint32_t i = t; i < m; i += 256u) {
    const uint4 v = __ldcg(&mb.list_in[i]);  // (a, c, c', x)
    const bool ins = v.w != 0xFFFFFFFFu;      // (not a migrant that left)
    dS += (int)(v.w < B0) - (int)(v.x < B0);
    dC += (int)(ins && v.y < B0) - (int)(v.z < B0);
    auto push = [&](int k, uint32_t p, int w) {
      const uint32_t q = atomicAdd(&s_ne[k], 1u);
      if (q < kMergeEv) s_ev[k][q] = make_int2((int)p, w);
    };
    if (v.w - B0 < kMergeSpan) push(0, v.w, 1);   // insertion point: stayers from x on
    if (v.x - B0 < kMergeSpan) push(0, v.x, -1);  // mover slot: stayers from a on
    if (ins && v.y - B0 < kMergeSpan) push(1, v.y, 1);  // new key: cells above c
    if (v.z - B0 < kMergeSpan) push(1, v.z, -1);  // previous key: cells above c'
  }
  {
    const int2 s2 = block_sum2(dS, dC, red2);
    dS = s2.x;
    dC = s2.y;
  }
  const uint32_t neS = s_ne[0], neC = s_ne[1];
  const bool spill = neS > kMergeEv || neC > kMergeEv;  // (clustered movers: exact slow path)
  // stayers: new slot s + #{x <= s} - #{a <= s}; movers are skipped
#pragma unroll
  for (int u = 0; u < kMergeItems; ++u) {
    const uint32_t s = B0 + u * 256u + t;
    if (s >= n) continue;
    int d = dS;
    bool mover = false;
    if (!spill) {
      for (uint32_t k = 0; k < neS; ++k) {
        const int2 ev = s_ev[0][k];
        if ((uint32_t)ev.x <= s) d += ev.y;
        mover |= ev.y < 0 && (uint32_t)ev.x == s;
      }
    } else {
      d = 0;
      for (uint32_t i = 0; i < m; ++i) {
        const uint4 v = __ldcg(&mb.list_in[i]);
        d += (int)(v.w <= s) - (int)(v.x <= s);
        mover |= v.x == s;
      }
    }
    if (mover) continue;
    const uint32_t j = base + (uint32_t)((int)s + d);
    // one radius: .w carries the old slot, and nothing on that path reads
    // perm (dem_get_grid extracts it from .w), so it is not written
    if (sw) P[u].w = __uint_as_float(s);
    else perm[j] = s;
    pos_sorted[j] = P[u];
  }
  // offsets, in place, only where the shift is not zero
  if (B0 <= c_hi && !(dC == 0 && neC == 0)) {
#pragma unroll
    for (int u = 0; u < kMergeItems; ++u) {
      const uint32_t c = B0 + u * 256u + t;
      if (c > c_hi || c < c_lo) continue;
      int d = dC;
      if (!spill) {
        for (uint32_t k = 0; k < neC; ++k) {
          const int2 ev = s_ev[1][k];
          if ((uint32_t)ev.x < c) d += ev.y;
        }
      } else {
        d = 0;
        for (uint32_t i = 0; i < m; ++i) {
          const uint4 v = __ldcg(&mb.list_in[i]);
          d += (int)(v.w != 0xFFFFFFFFu && v.y < c) - (int)(v.z < c);
        }
      }
      if (d != 0) off[c] = (uint32_t)((int)__ldcs(&off[c]) + d);
    }
  }
  // movers b, b + grid, ...: r_i + x_i - #{a_j < x_i}, counted block-wide
  for (uint32_t i = b; i < m; i += mgrid) {
    const uint4 mi = __ldcg(&mb.list_in[i]);
    if (mi.w == 0xFFFFFFFFu) continue;  // (block-uniform) a migrant that left: no insertion
    int r = 0;
    for (uint32_t jj = t; jj < m; jj += 256u) {
      const uint4 v = __ldcg(&mb.list_in[jj]);
      // (c, arrival from the left first, slot) order of the insertions
      const bool vl = v.z == 0xFFFFFFFEu, ml = mi.z == 0xFFFFFFFEu;
      r += (int)(v.w != 0xFFFFFFFFu &&
                 (v.y < mi.y || (v.y == mi.y && (vl > ml || (vl == ml && v.x < mi.x))))) -
           (int)(v.x < mi.w);
    }
    r = block_sum(r, red[0]);
    if (t == 0) {
      const uint32_t j = base + (uint32_t)(r + (int)mi.w);
      float4 Pm = __ldg(&pos_in[mi.x]);
      if (sw) Pm.w = __uint_as_float(mi.x);
      else perm[j] = mi.x;
      pos_sorted[j] = Pm;
    }
  }
}

// ----------------------------------------------------------- k_sweep -------

// Eqs. 2-10 for one contact seen from particle i (R1 orientation). Returns
// the force on i, Tc = n x F_t (the torque is r_i Tc, Eq. 3) and the new δ_t.
__device__ __forceinline__ void pair_practical(f3 n, float delta, float Rs, float ms, f3 v,
                                               f3 rw, f3 dold, float Cn, float Ct, float alpha,
                                               float mu, float dt, uint32_t flags, f3& F, f3& Tc,
                                               f3& dnew) {
  const float s = fsqrt(delta * Rs);  // Eqs. 8-9 share sqrt(|δ_n| / (r_i^-1 + r_j^-1))
  const float kn = Cn * s, kt = Ct * s;
  const float eta = alpha * fsqrt(kn * ms);  // Eq. 10
  const float vn = dot(v, n);
  const f3 c = cross(rw, n);
  const f3 vt = mk((v.x - vn * n.x) + c.x, (v.y - vn * n.y) + c.y, (v.z - vn * n.z) + c.z);  // Eq. 6
  const float p = dot(dold, n);
  dnew = mk((dold.x - p * n.x) + vt.x * dt, (dold.y - p * n.y) + vt.y * dt,
            (dold.z - p * n.z) + vt.z * dt);  // Eq. 7
  const float knd = kn * delta;
  f3 Fn = mk(-knd * n.x - eta * (vn * n.x), -knd * n.y - eta * (vn * n.y),
             -knd * n.z - eta * (vn * n.z));  // Eq. 4, normal
  f3 Ft = mk(-kt * dnew.x - eta * vt.x, -kt * dnew.y - eta * vt.y,
             -kt * dnew.z - eta * vt.z);  // Eq. 4, tangential
  // DEM_F_CLAMP_FN (R3 flag): no tensile normal force. knd and η (v·n) are
  // the same numbers from either side of the pair, so the decision is too (P11)
  if ((flags & 2u) && knd + eta * vn < 0.f) Fn = mk(0.f, 0.f, 0.f);
  const float fn = fsqrt(dot(Fn, Fn));
  const float ft2 = dot(Ft, Ft);
  const float lim = mu * fn;
  if (ft2 > lim * lim) {  // Eq. 5: |F_t| > μ|F_n|
    // (ft2 held at >= FLT_MIN: the .ftz sqrt would flush a subnormal ft2 to 0
    // and lim * rcp(0) be inf, or NaN for lim = 0 — μ = 0 or a clamped F_n)
    const float sc = lim * frcp(fsqrt(fmaxf(ft2, 1.17549435e-38f)));
    Ft = mk(Ft.x * sc, Ft.y * sc, Ft.z * sc);
    if ((flags & 1u) && kt > 0.f) {  // DEM_F_TRUNCATE_DT (R4)
      const float ik = frcp(kt);
      dnew = mk(-(Ft.x + eta * vt.x) * ik, -(Ft.y + eta * vt.y) * ik, -(Ft.z + eta * vt.z) * ik);
    }
  }
  F = mk(Fn.x + Ft.x, Fn.y + Ft.y, Fn.z + Ft.z);  // Eq. 2
  Tc = cross(n, Ft);                               // Eq. 3 (without r_i)
}

// Eq. 1 in the SDK sign convention (R1), u = v_j - v_i.
__device__ __forceinline__ f3 pair_simple(f3 n, float delta, f3 u, float ksp, float kda,
                                          float ksh) {
  const float un = dot(u, n);
  const float kd = ksp * delta;
  return mk((-kd * n.x + kda * u.x) + ksh * (u.x - un * n.x),
            (-kd * n.y + kda * u.y) + ksh * (u.y - un * n.y),
            (-kd * n.z + kda * u.z) + ksh * (u.z - un * n.z));
}

// Exact contact predicate of R14 in fp64 (no contraction: __dmul_rn/__dadd_rn).
__device__ __forceinline__ double exact_d2(float4 P, float4 Q) {
  const double dx = (double)Q.x - (double)P.x, dy = (double)Q.y - (double)P.y,
               dz = (double)Q.z - (double)P.z;
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Contact predicate (R14): fp32 decides outside a ±16u band around S², the
// exact fp64 expression inside it (|d²₃₂ - d²| <= 5u d², |S²₃₂ - S²| <= 3u S²).
__device__ __forceinline__ bool in_contact(float4 P, float4 Q) {
  const float dxf = Q.x - P.x, dyf = Q.y - P.y, dzf = Q.z - P.z;
  const float d2f = dxf * dxf + dyf * dyf + dzf * dzf;
  const float Sf = P.w + Q.w;
  const float S2f = Sf * Sf;
  if (d2f >= S2f * 1.00000095367431640625f) return false;  // (1 + 16u) S²: clearly apart
  if (d2f <= S2f * 0.99999904632568359375f) return true;   // (1 - 16u) S²: clearly touching
  const double S = (double)P.w + (double)Q.w;
  return exact_d2(P, Q) < __dmul_rn(S, S);
}

// Geometry of a contact from the fp32 values: n (fp32, i -> j) and the
// overlap δ = S - D evaluated as (S² - d²)/(S + D) with the numerator in fp64
// (S² is exact in fp64; d² has the fixed order of R14) — the cancellation of
// S - D is in exact-ish fp64, the division in fp32. Symmetric in (i, j).
// Returns false for coincident centres (R18): d² = 0, or d² below FLT_MIN,
// whose fp32 value the .ftz square root would flush (|Δ| < 1.1e-19 m, only
// reachable for centres within ~1e-12 m of the coordinate origin; DESIGN R18).
__device__ __forceinline__ bool contact_geometry(float4 P, float4 Q, f3& n, float& delta) {
  const double d2 = exact_d2(P, Q);
  if (!(d2 >= 1.17549435082228751e-38)) return false;
  const double S = (double)P.w + (double)Q.w;
  const float num = (float)__dsub_rn(__dmul_rn(S, S), d2);
  const float D = fsqrt((float)d2);
  delta = fmaxf(num * frcp(__fadd_rn((float)S, D)), 0.f);
  const float invD = frcp(D);
  n = mk((Q.x - P.x) * invD, (Q.y - P.y) * invD, (Q.z - P.z) * invD);
  return true;
}

struct Own {  // the particle of a sorted slot, as one contact evaluation needs it
  float4 P, V, W;  // (x, r), (v, m), (ω, id bits)
};

// Steps 7 for one particle pair (i owner, j partner): practical model with
// history. `dold` is δ_t,old of the pair (0 if new). Returns F on i, Tc.
template <bool MAT = true>
__device__ __forceinline__ void eval_pair_practical(const Own& o, float4 Q, float4 VQ, float4 WQ,
                                                    f3 n, float delta, f3 dold, const DevPhys& ph,
                                                    f3& Fc, f3& Tc, f3& dnew) {
  const float Rs = frcp(__fadd_rn(frcp(o.P.w), frcp(Q.w)));
  const float ms = frcp(__fadd_rn(frcp(o.V.w), frcp(VQ.w)));
  const f3 v = mk(o.V.x - VQ.x, o.V.y - VQ.y, o.V.z - VQ.z);
  // r_i ω_i + r_j ω_j with no contraction, so both sides round it identically (P11)
  const f3 rw = mk(__fadd_rn(__fmul_rn(o.P.w, o.W.x), __fmul_rn(Q.w, WQ.x)),
                   __fadd_rn(__fmul_rn(o.P.w, o.W.y), __fmul_rn(Q.w, WQ.y)),
                   __fadd_rn(__fmul_rn(o.P.w, o.W.z), __fmul_rn(Q.w, WQ.z)));
  float Cn = ph.Cn, Ct = ph.Ct, alpha = ph.alpha, mu = ph.mu;
  if (MAT && ph.nmat > 1) {  // C_k(i, j), α(i, j), μ(i, j) of the two materials (Eqs. 5, 8-10)
    const uint32_t mi = __float_as_uint(o.W.w) >> kMatShift, mj = __float_as_uint(WQ.w) >> kMatShift;
    const float4 c = __ldg(&ph.mat[mi * ph.nmat + mj]);
    Cn = c.x, Ct = c.y, alpha = c.z, mu = c.w;
  }
  pair_practical(n, delta, Rs, ms, v, rw, dold, Cn, Ct, alpha, mu, ph.dt, ph.flags, Fc, Tc, dnew);
}

// Plate k (R23) against particle P = (x, r): the rectangle's point closest
// to the centre, in fp64 on the fp32 plate numbers (centre c, unit normal n,
// unit axis u, half-lengths a, b along u and v = n x u). Returns (unit vector
// from the centre to that point, δ = r - distance) when in contact, w <= 0
// when not, w = NaN for a centre on the plate. Out of line: plates are few
// and rarely touched, so the common path keeps its registers.
__device__ __noinline__ float4 plate_contact(const float* __restrict__ pl, float4 P) {
  if (fabsf((P.x - pl[0]) * pl[3] + (P.y - pl[1]) * pl[4] + (P.z - pl[2]) * pl[5]) >
      P.w * 1.0001f + 1e-6f * (fabsf(P.x) + fabsf(P.y) + fabsf(P.z)) + 1e-30f)
    return make_float4(0.f, 0.f, 0.f, -1.f);  // conservative fp32 reject: far from the plane
  // the exact fp64 expression of R23, evaluated in a fixed order without
  // contraction (the oracle's order), so contact decisions are bit-identical
  const double c[3] = {pl[0], pl[1], pl[2]}, n[3] = {pl[3], pl[4], pl[5]};
  const double u[3] = {pl[6], pl[7], pl[8]};
  const double v[3] = {__dsub_rn(__dmul_rn(n[1], u[2]), __dmul_rn(n[2], u[1])),
                       __dsub_rn(__dmul_rn(n[2], u[0]), __dmul_rn(n[0], u[2])),
                       __dsub_rn(__dmul_rn(n[0], u[1]), __dmul_rn(n[1], u[0]))};
  const double x[3] = {(double)P.x, (double)P.y, (double)P.z};
  double du = 0.0, dv = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    du = __dadd_rn(du, __dmul_rn(__dsub_rn(x[a], c[a]), u[a]));
    dv = __dadd_rn(dv, __dmul_rn(__dsub_rn(x[a], c[a]), v[a]));
  }
  const double qu = fmin(fmax(du, -(double)pl[9]), (double)pl[9]);
  const double qv = fmin(fmax(dv, -(double)pl[10]), (double)pl[10]);
  double e[3], d2 = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    e[a] = __dsub_rn(__dadd_rn(__dadd_rn(c[a], __dmul_rn(qu, u[a])), __dmul_rn(qv, v[a])), x[a]);
    d2 = __dadd_rn(d2, __dmul_rn(e[a], e[a]));
  }
  const double dist = __dsqrt_rn(d2), r = (double)P.w;
  if (!(r > dist)) return make_float4(0.f, 0.f, 0.f, -1.f);
  if (dist == 0.0) return make_float4(0.f, 0.f, 0.f, __int_as_float(0x7fc00000));
  return make_float4((float)__ddiv_rn(e[0], dist), (float)__ddiv_rn(e[1], dist),
                     (float)__ddiv_rn(e[2], dist), (float)__dsub_rn(r, dist));
}


// The step's outputs (next state, its key and history) are not read again in
// this step: DEM_OUT_CS stores them evict-first in L2 (st.global.cs), so
// they do not displace the neighbour state the contact rounds re-read.
#ifndef DEM_OUT_CS
#define DEM_OUT_CS 0
#endif
template <class T>
__device__ __forceinline__ void st_out(T* p, T v) {
  if (DEM_OUT_CS) __stcs(p, v);
  else *p = v;
}

// Step 8 + step 1 + next step 2 for one particle (shared by both sweeps):
// walls, integration, state write at slot j, next CM and its counting rank.
// The outputs go to slot oj = j - (first owned sorted slot): the owned
// particles of the next step are dense from 0.
// MAT: the handle has material tables or plates (k_force is instantiated both
// ways so that the common case carries neither).
template <int MODEL, bool DIAG, bool MAT = true, class LookupFn>
__device__ __forceinline__ void finish_particle(const StepBuffers& b, const DevGrid& g,
                                                const DevPhys& ph, uint32_t N, uint32_t K,
                                                uint32_t oj, const Own& o, f3 F, f3 T,
                                                uint32_t ncnt, bool overflow, LookupFn lookup,
                                                uint32_t sk_known = 0xFFFFFFFFu) {
  const uint32_t j = oj;  // output slot
  // this step's SCM at j (merge re-sort): the key of the sorted position itself
  // (the sort ordered these very coordinates by it), so no SCM array is kept
  const uint32_t sk = !b.mv.list_out ? 0u : sk_known != 0xFFFFFFFFu ? sk_known
                                                                    : cell_key(g, o.P.x, o.P.y, o.P.z);
  const float ri = o.P.w, mi = o.V.w;
  const uint32_t my_id = __float_as_uint(o.W.w) & (MAT ? ph.idmask : 0xFFFFFFFFu);
  // step 8: walls -x,+x,-y,+y,-z,+z as particles of infinite radius (R11)
  const float xs[3] = {o.P.x, o.P.y, o.P.z};
  // conservative fp32 prefilter: only particles within r (+ rounding margin)
  // of a face evaluate the exact fp64 wall predicate
  bool near_wall = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float m = ri + 1e-6f * (fabsf(xs[a]) + ri) + 1e-30f;
    near_wall |= (xs[a] - (float)g.lo[a] < m) | ((float)g.hi[a] - xs[a] < m);
  }
  // one wall contact (a face or a plate): Eqs. 2-10 with R* = r_i, m* = m_i,
  // v_j = ω_j = 0 (R11), the wall coefficients (per material if tabulated)
  auto wall_contact = [&](f3 n, float delta, uint32_t pid) {
    if (MODEL == 0) {
      const f3 rwi = mk(__fmul_rn(ri, o.W.x), __fmul_rn(ri, o.W.y), __fmul_rn(ri, o.W.z));
      f3 Fc, Tc, dnew;
      float4 c = make_float4(ph.wCn, ph.wCt, ph.walpha, ph.wmu);
      if (MAT && ph.nmat > 1) c = __ldg(&ph.wmat[__float_as_uint(o.W.w) >> kMatShift]);
      pair_practical(n, delta, ri, mi, mk(o.V.x, o.V.y, o.V.z), rwi, lookup(pid), c.x, c.y, c.z,
                     c.w, ph.dt, ph.flags, Fc, Tc, dnew);
      F = mk(F.x + Fc.x, F.y + Fc.y, F.z + Fc.z);
      T = mk(T.x + ri * Tc.x, T.y + ri * Tc.y, T.z + ri * Tc.z);
      if (ncnt < K) {
        st_out(&b.hist_out[hix(j, ncnt, K)], make_float4(dnew.x, dnew.y, dnew.z, __uint_as_float(pid)));
        ++ncnt;
      } else {
        overflow = true;
      }
    } else {
      const f3 Fc = pair_simple(n, delta, mk(-o.V.x, -o.V.y, -o.V.z), ph.ksp, ph.kda, ph.ksh);
      F = mk(F.x + Fc.x, F.y + Fc.y, F.z + Fc.z);
    }
  };
#pragma unroll
  for (int w = 0; w < 6; ++w) {
    if (!near_wall) break;
    const int a = w >> 1;
    const bool hi = (w & 1) != 0;
    const double dist = hi ? (g.hi[a] - (double)xs[a]) : ((double)xs[a] - g.lo[a]);
    if (!((double)ri > dist)) continue;
    f3 n = mk(0.f, 0.f, 0.f);
    if (a == 0) n.x = hi ? 1.f : -1.f;
    if (a == 1) n.y = hi ? 1.f : -1.f;
    if (a == 2) n.z = hi ? 1.f : -1.f;
    wall_contact(n, (float)((double)ri - dist), kWallPid0 + (uint32_t)w);
  }
  // plates (R23), in the order given; geometry out of line (rarely taken)
  for (uint32_t k = 0; MAT && k < ph.nplates; ++k) {
    const float4 c = plate_contact(ph.plates + 12 * k, o.P);
    if (!(c.w > 0.f) && !isnan(c.w)) continue;  // no contact
    if (isnan(c.w)) {  // centre on the plate: no direction (R18)
      raise_error(b.err, 9u, j, my_id);
      continue;
    }
    wall_contact(mk(c.x, c.y, c.z), c.w, kWallPid0 + 6u + k);
  }
  if (overflow) raise_error(b.err, 6u, j, my_id);
  if (MODEL == 0) st_out(&b.cnt_out[j], ncnt);
  if (DIAG) {
    b.F_out[j] = make_float4(F.x, F.y, F.z, 0.f);
    b.T_out[j] = make_float4(T.x, T.y, T.z, 0.f);
  }
  // step 1 (next iteration): semi-implicit Euler (R9)
  const float dt = ph.dt;
  const float im = frcp(mi);
  const float ax = F.x * im + ph.g[0], ay = F.y * im + ph.g[1], az = F.z * im + ph.g[2];
  const float vx = o.V.x + ax * dt, vy = o.V.y + ay * dt, vz = o.V.z + az * dt;
  const float x = o.P.x + vx * dt, y = o.P.y + vy * dt, z = o.P.z + vz * dt;
  float wx = o.W.x, wy = o.W.y, wz = o.W.z;
  if (MODEL == 0) {
    const float iI = frcp(0.4f * mi * ri * ri);
    wx = o.W.x + (T.x * iI) * dt;
    wy = o.W.y + (T.y * iI) * dt;
    wz = o.W.z + (T.z * iI) * dt;
  }
  st_out(&b.pos_out[j], make_float4(x, y, z, ri));
  st_out(&b.vel_out[j], make_float4(vx, vy, vz, mi));
  st_out(&b.omg_out[j], make_float4(wx, wy, wz, o.W.w));
  const bool finite = isfinite(x) && isfinite(y) && isfinite(z) && isfinite(vx) &&
                      isfinite(vy) && isfinite(vz) && isfinite(wx) && isfinite(wy) &&
                      isfinite(wz);
  uint32_t k2 = 0, xf = 0;  // (xf: slab exchange flags)
  if (!finite) {
    raise_error(b.err, 7u, j, my_id);
  } else {
    const double rd = (double)ri;
    if ((double)x < g.lo[0] - rd || (double)x > g.hi[0] + rd || (double)y < g.lo[1] - rd ||
        (double)y > g.hi[1] + rd || (double)z < g.lo[2] - rd || (double)z > g.hi[2] + rd)
      raise_error(b.err, 8u, j, my_id);
    k2 = cell_key(g, x, y, z);  // step 2 of the next step: CM of the new position
    if (g.slab) {
      // slab exchange flags: leaving the owned planes = a
      // migrant to the left (bit 0) or right (bit 1) neighbour. It keeps its
      // key: it lies in this rank's ghost plane, where this rank's boundary
      // particles need it as a neighbour next step (the receiver, which did
      // not own it when it packed its plane, cannot send it back in time).
      const int cz = cell_coord(z, g.lo[2], g.inv_h, g.nz_global);
      uint32_t f = 0;
      if (cz < g.z0) f |= 1u;
      if (cz >= g.z1) f |= 2u;
      b.flags[j] = f;
      xf = f;
    }
  }
  if (g.slab) {
    // the pack's tile counts per category (tiles of kXTile output slots):
    // one atomic per (warp, tile, category) with flagged lanes, so the pack
    // needs no counting pass (most warps have none: boundary planes only)
    const uint32_t act = __activemask();
    const uint32_t tile = j / kXTile;
    const uint32_t peers = __match_any_sync(act, tile);
    const uint32_t leader = __ffs(peers) - 1;
    const uint32_t any = __ballot_sync(act, xf != 0u) & peers;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t m = __ballot_sync(act, (xf >> q) & 1u) & peers;
      if (m && lane_id() == leader) atomicAdd(&b.xtc[(uint32_t)q * b.xntiles + tile], __popc(m));
    }
    // per-tile sum; the first contribution to a tile counts the tile (the
    // pack's last writing block publishes)
    if (any && lane_id() == leader &&
        atomicAdd(&b.xtc[4u * b.xntiles + tile], __popc(any)) == 0u)
      atomicAdd(&b.xtc[5u * b.xntiles], 1u);
  }
  st_out(&b.key_out[j], k2);
  if (b.mv.list_out) {  // merge re-sort: list the particles that change cell (warp-aggregated)
    const uint32_t act = __activemask();
    const uint32_t mv = __ballot_sync(act, k2 != sk);
    if (mv) {
      const uint32_t leader = __ffs(mv) - 1;
      uint32_t base = 0;
      if (lane_id() == leader) base = atomicAdd(b.mv.n_out, (uint32_t)__popc(mv));
      base = __shfl_sync(act, base, leader);
      const uint32_t idx = base + (uint32_t)__popc(mv & lanemask_lt());
      if (k2 != sk && idx < b.mv.cap) {
        // slot, new key, previous key and the insertion point among this
        // step's order (these offsets are the next step's previous ones;
        // slab ranks: relative to the owned particles' first sorted slot). A
        // migrant leaves the owned particles: insertion point 0xFFFFFFFF
        const uint32_t gl = b.gl_base;
        const uint32_t x = (xf & 3u) ? 0xFFFFFFFFu
                                     : min(max(j, __ldg(&b.off[k2]) - gl), __ldg(&b.off[k2 + 1]) - gl);
        b.mv.list_out[idx] = make_uint4(j, k2, sk, x);
      }
    }
  } else {
    b.prank[j] = count_into_cell(b.count, k2);  // counted into its cell for the next sort
  }
}

#if DEM_ABLATIONS  // (built into libdem_ablations.so only)
// ---- ablation: one thread per sorted particle for the whole step ----------
// The paper's mapping ("Assign the i-th thread to the SCM[i]-th
// particle"): each thread loops over its candidates and evaluates its own
// contacts, so a warp idles on the lanes without a contact (§6's "quarter").
template <int MODEL, bool DIAG, bool MAT>
__global__ void __launch_bounds__(128) k_sweep_tpp(StepBuffers b, DevGrid g, DevPhys ph,
                                                   uint32_t N, uint32_t K) {
  pdl_enter();
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t jlo = __ldg(&b.off[g.own_c0]), jhi = __ldg(&b.off[g.own_c1]);
  const uint32_t j = jlo + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= jhi) return;
  const uint32_t s = __ldg(&b.perm[j]);
  Own o;
  o.P = __ldg(&b.pos_sorted[j]);
  o.V = __ldg(&b.vel_in[s]);
  o.W = __ldg(&b.omg_in[s]);
  const uint32_t n_old = MODEL == 0 ? __ldg(&b.cnt_in[s]) : 0u;
  auto lookup = [&](uint32_t pid) -> f3 {
    for (uint32_t k = 0; k < n_old; ++k) {
      const float4 h = __ldg(&b.hist_in[hix(s, k, K)]);
      if (__float_as_uint(h.w) == pid) return mk(h.x, h.y, h.z);
    }
    return mk(0.f, 0.f, 0.f);
  };
  const int cx = cell_coord(o.P.x, g.lo[0], g.inv_h, g.nx);
  const int cy = cell_coord(o.P.y, g.lo[1], g.inv_h, g.ny);
  const int cz = cell_coord(o.P.z, g.lo[2], g.inv_h, g.nz_global) - g.zlo;
  f3 F = mk(0.f, 0.f, 0.f), T = mk(0.f, 0.f, 0.f);
  uint32_t ncnt = 0;
  bool overflow = false;
  const int xa = cx > 0 ? cx - 1 : 0;
  const int xb = cx < g.nx - 1 ? cx + 1 : g.nx - 1;
  for (int dz = -1; dz <= 1; ++dz) {
    const int z = cz + dz;
    if (z < 0 || z >= g.nz) continue;
    for (int dy = -1; dy <= 1; ++dy) {
      const int y = cy + dy;
      if (y < 0 || y >= g.ny) continue;
      const uint32_t row = ((uint32_t)z * (uint32_t)g.ny + (uint32_t)y) * (uint32_t)g.nx;
      const uint32_t t0 = __ldg(&b.off[row + xa]);
      const uint32_t t1 = __ldg(&b.off[row + xb + 1]);
      for (uint32_t t = t0; t < t1; ++t) {
        if (t == j) continue;
        const float4 Q = __ldg(&b.pos_sorted[t]);
        if (!in_contact(o.P, Q)) continue;
        f3 n;
        float delta;
        if (!contact_geometry(o.P, Q, n, delta)) {
          raise_error(b.err, 9u, j, __float_as_uint(o.W.w) & ph.idmask);
          continue;
        }
        const uint32_t q = __ldg(&b.perm[t]);
        const float4 VQ = __ldg(&b.vel_in[q]);
        if (MODEL == 0) {
          const float4 WQ = __ldg(&b.omg_in[q]);
          const uint32_t pid = __float_as_uint(WQ.w) & ph.idmask;
          f3 Fc, Tc, dnew;
          eval_pair_practical<MAT>(o, Q, VQ, WQ, n, delta, lookup(pid), ph, Fc, Tc, dnew);
          F = mk(F.x + Fc.x, F.y + Fc.y, F.z + Fc.z);
          T = mk(T.x + o.P.w * Tc.x, T.y + o.P.w * Tc.y, T.z + o.P.w * Tc.z);
          if (ncnt < K) {
            b.hist_out[hix(j - jlo, ncnt, K)] =
                make_float4(dnew.x, dnew.y, dnew.z, __uint_as_float(pid));
            ++ncnt;
          } else {
            overflow = true;
          }
        } else {
          const f3 u = mk(VQ.x - o.V.x, VQ.y - o.V.y, VQ.z - o.V.z);
          const f3 Fc = pair_simple(n, delta, u, ph.ksp, ph.kda, ph.ksh);
          F = mk(F.x + Fc.x, F.y + Fc.y, F.z + Fc.z);
        }
      }
    }
  }
  finish_particle<MODEL, DIAG, MAT>(b, g, ph, N, K, j - jlo, o, F, T, ncnt, overflow, lookup);
}

#endif  // DEM_ABLATIONS

// ---- default path: k_detect (steps 5-6) then k_force (steps 7-8, 1) -------
// k_detect: one light thread per sorted particle scans its 27-cell candidates
// (Eq. 12: 9 contiguous slot ranges of sorted positions, row bounds loaded per
// z-plane) with the exact predicate (R14) and writes its contact list
// clist[k*N + j] = t (each partner's sorted slot, in candidate order =
// ascending sorted slot). Few registers, so the SM keeps many warps in flight
// to hide the neighbour-row latency.
// Owned sorted slots [jlo, jhi): single GPU all N slots (no memory access on
// the critical path), slab mode [off[own_c0], off[own_c1]).
__device__ __forceinline__ void owned_range(const StepBuffers& b, const DevGrid& g, uint32_t N,
                                            uint32_t& jlo, uint32_t& jhi) {
  if (g.slab) {
    jlo = __ldg(&b.off[g.own_c0]);
    jhi = __ldg(&b.off[g.own_c1]);
  } else {
    jlo = 0u;
    jhi = N;
  }
}

// One scan of the 27-cell candidates of sorted slot j (9 row ranges, bounds
// loaded per z-plane). FAST: the fp32 decision r = d² - S² < 0 only, with
// `amb` raised (>= 0) when some candidate lies inside the ±16u band of R14 —
// the caller then rescans with EXACT, which settles band candidates in fp64.
// fl(d² - S²) keeps the sign of d² - S², and outside the band the fp32 and
// exact decisions agree (in_contact's bound), so both scans give one list.
// MONO: all radii equal, S2c = fl((2r)²) (what the general expression gives
// for every pair); a candidate is decided with the EXACT scan's own fp32
// thresholds — touching below S²(1 - 16u), apart from S²(1 + 16u) on — and one
// in between sets `amb` to 0, so outside the band both scans decide alike and
// a non-touching candidate costs a single compare.
// MONO also means pos_sorted[t].w holds the old slot SCCM[t] (b.sw_r): the
// list stores that (what k_force reads partner state by) and the radius is
// b.sw_r.
// The list goes to `out` with stride `ostride` (k_detect: clist + j, N; the
// fused sweep: its warp's shared-memory list, [k][lane]).
#ifndef DEM_DETECT_FLAT
#define DEM_DETECT_FLAT 3
#endif
// fused sweep (SMEM): each plane's 3 rows scanned as one run, kDetectFlat
// candidate loads per trip (C3 -4%; k_detect's 32-register threads spill
// with it, +27% there — profiles/r2_history.md #26)
constexpr int kDetectFlat = DEM_DETECT_FLAT;
// the per-row candidate loop with per-particle radii unrolled by six:
// several candidate loads in flight per trip (C5 k_detect -6%, r2 history #37)
#ifndef DEM_ROW_UNROLL
#define DEM_ROW_UNROLL 6
#endif
constexpr int kRowUnroll = DEM_ROW_UNROLL;
// per-particle radii: the fast scan's band test (the EXACT scan's own
// thresholds S²(1 ± 16u)) inside the hit branch, as with one radius, instead
// of a running max of 16u S² - |d² - S²| over every candidate
#ifndef DEM_DETECT_BAND_BRANCH
#define DEM_DETECT_BAND_BRANCH 1
#endif
constexpr bool kDetectBandBranch = DEM_DETECT_BAND_BRANCH != 0;
// the dense configuration's (PRED) runs: five loads per trip (C3 -3%, r2 history #33)
#ifndef DEM_DETECT_FLAT_DENSE
#define DEM_DETECT_FLAT_DENSE 5
#endif
constexpr int kDetectFlatDense = DEM_DETECT_FLAT_DENSE;
// PRED (fused sweep, dense configuration): a hit handled by predicated
// instructions instead of a branch — with ~10 contacts per particle some lane
// of the warp hits almost every candidate index, so the branch was always
// taken (C2 -5%, C3 -1%; the light bed C4 +2%: r2 history #29)
template <bool EXACT, bool MONO = false, bool SMEM = false, bool PRED = false,
          int FLAT = kDetectFlat>
__device__ __forceinline__ uint32_t detect_scan(const StepBuffers& b, const DevGrid& g, float4 P,
                                                int cx, int cy, int cz, uint32_t j,
                                                uint32_t* out, uint32_t ostride,
                                                uint32_t K, float& amb, float S2c = 0.f) {
  const uint32_t xa = cx > 0 ? (uint32_t)cx - 1u : 0u;
  const uint32_t xb = cx < g.nx - 1 ? (uint32_t)cx + 1u : (uint32_t)g.nx - 1u;
  const uint32_t nxy = (uint32_t)g.nx * (uint32_t)g.ny;
  uint32_t npair = 0;
  // MONO fast scan: candidates with d² < S²(1 + 16u) take the hit branch, and
  // those of them above S²(1 - 16u) are in the band (the EXACT scan's own
  // thresholds), so a non-touching candidate costs one compare
  const float S2lo = S2c * 0.99999904632568359375f, S2hi = S2c * 1.00000095367431640625f;
  constexpr int kFlat = FLAT;
  if (!EXACT && MONO && SMEM && kFlat > 1) {
    // the plane's 3 rows as one flattened run u = 0..n0+n1+n2 (the same
    // candidate order), kFlat candidate loads in flight per iteration
#pragma unroll 1
    for (int dz = -1; dz <= 1; ++dz) {
      const int z = cz + dz;
      if (z < 0 || z >= g.nz) continue;
      uint32_t t0[3], t1[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int y = cy + r - 1;
        const bool in = y >= 0 && y < g.ny;
        const uint32_t row = (uint32_t)z * nxy + (uint32_t)(in ? y : 0) * (uint32_t)g.nx;
        t0[r] = in ? __ldg(&b.off[row + xa]) : 0u;
        t1[r] = in ? __ldg(&b.off[row + xb + 1]) : 0u;
      }
      const uint32_t c1 = t1[0] - t0[0], c2 = c1 + (t1[1] - t0[1]), nt = c2 + (t1[2] - t0[2]);
      const uint32_t b0 = t0[0], b1 = t0[1] - c1, b2 = t0[2] - c2;  // t = u + b(row of u)
#pragma unroll 1
      for (uint32_t u = 0; u < nt; u += (uint32_t)(kFlat > 1 ? kFlat : 1)) {
        constexpr int U = kFlat > 1 ? kFlat : 1;
        float4 Q[U];
        uint32_t tt[U];
#pragma unroll
        for (int v = 0; v < U; ++v) {
          const uint32_t uu = u + (uint32_t)v;
          tt[v] = uu + (uu < c1 ? b0 : uu < c2 ? b1 : b2);
          Q[v] = uu < nt ? __ldg(&b.pos_sorted[tt[v]]) : make_float4(3.0e38f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int v = 0; v < U; ++v) {
          const float dx = Q[v].x - P.x, dy = Q[v].y - P.y, dz2 = Q[v].z - P.z;
          const float d2 = dx * dx + dy * dy + dz2 * dz2;
          if (PRED) {
            const bool hit = d2 < S2hi && tt[v] != j;
            amb = hit && d2 > S2lo ? 0.f : amb;
            if (hit && npair < K) out[npair * ostride] = __float_as_uint(Q[v].w);
            npair += hit ? 1u : 0u;
          } else if (d2 < S2hi && tt[v] != j) {
            asm volatile("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.f32 %0, 0f00000000, %3, p;}"
                         : "=f"(amb) : "f"(d2), "f"(S2lo), "f"(amb));
            if (npair < K) {
              if (SMEM) *out = __float_as_uint(Q[v].w);
              else __stcg(out, __float_as_uint(Q[v].w));
            }
            out += ostride;
            ++npair;
          }
        }
      }
    }
    return npair;
  }
#pragma unroll 1
  for (int dz = -1; dz <= 1; ++dz) {
    const int z = cz + dz;
    if (z < 0 || z >= g.nz) continue;
    uint32_t t0[3], t1[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {  // the plane's 6 row bounds in flight together
      const int y = cy + r - 1;
      const bool in = y >= 0 && y < g.ny;
      const uint32_t row = (uint32_t)z * nxy + (uint32_t)(in ? y : 0) * (uint32_t)g.nx;
      t0[r] = in ? __ldg(&b.off[row + xa]) : 0u;
      t1[r] = in ? __ldg(&b.off[row + xb + 1]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll (MONO ? 1 : kRowUnroll)
      for (uint32_t t = t0[r]; t < t1[r]; ++t) {
        float4 Q = __ldg(&b.pos_sorted[t]);
        const uint32_t qs = MONO ? __float_as_uint(Q.w) : t;  // what the list stores
        if (MONO) Q.w = b.sw_r;
        const float dx = Q.x - P.x, dy = Q.y - P.y, dz2 = Q.z - P.z;
        const float d2 = dx * dx + dy * dy + dz2 * dz2;
        const float S = P.w + Q.w;
        const float S2 = MONO ? S2c : S * S;
        bool hit;
        if (!EXACT && MONO) {
          hit = d2 < S2hi;  // (the band test is in the hit branch below)
        } else if (EXACT) {
          hit = d2 <= S2 * 0.99999904632568359375f;  // (1 - 16u) S²: clearly touching
          if (!hit && d2 < S2 * 1.00000095367431640625f) {  // inside the band: exact (R14)
            const double Sd = (double)P.w + (double)Q.w;
            hit = exact_d2(P, Q) < __dmul_rn(Sd, Sd);
          }
        } else if (kDetectBandBranch) {
          hit = d2 < S2 * 1.00000095367431640625f;  // as MONO, with this pair's S²
        } else {
          const float rr = d2 - S2;
          hit = rr < 0.f;
          amb = fmaxf(amb, fmaf(S2, 9.5367431640625e-7f, -fabsf(rr)));  // 16u S² - |r|
        }
        // only the middle row (y = cy) can hold slot j itself: the other two
        // rows skip the self test (r is unrolled, so it folds away there)
        if (hit && (r != 1 || t != j)) {
          if (!EXACT && (MONO || kDetectBandBranch)) {
            // band: the caller rescans exactly. volatile keeps the test in this
            // branch (if-converted, it would cost every candidate two instructions)
            const float lo = MONO ? S2lo : S2 * 0.99999904632568359375f;
            asm volatile("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.f32 %0, 0f00000000, %3, p;}"
                         : "=f"(amb) : "f"(d2), "f"(lo), "f"(amb));
          }
          if (npair < K) {
            if (SMEM) *out = qs;
            else __stcg(out, qs);
          }
          out += ostride;
          ++npair;
        }
      }
    }
  }
  return npair;
}

// k_detect: one light thread per sorted particle scans its 27-cell candidates
// (Eq. 12) with the exact predicate (R14) and writes its contact list
// clist[k*N + j] = t (each partner's sorted slot, in candidate order =
// ascending sorted slot). Few registers, so the SM keeps many warps in flight
// to hide the neighbour-row latency; the rare particle with a candidate in the
// fp32 uncertainty band rescans exactly.
// Two occupancy targets: 6 blocks of 256 (40 registers) and 8 (32 registers,
// a few spilled). The sparse lists of a light handle (c̄ <= 7: ~26 candidates,
// ~5 contacts) gain from the extra warps (C4: 160 -> 153 us); the dense C2/C3
// sets lose 3-8%, so the choice follows the k_force configuration.
#ifndef DEM_DETECT_MINB
#define DEM_DETECT_MINB 6
#endif
#ifndef DEM_DETECT_MINB_LIGHT
#define DEM_DETECT_MINB_LIGHT 8
#endif
// threads per k_detect block; the MINB targets above are in blocks of 256
#ifndef DEM_DETECT_TPB
#define DEM_DETECT_TPB 256
#endif
template <bool MONO, bool LIGHT = false>
__global__ void __launch_bounds__(DEM_DETECT_TPB, (LIGHT ? DEM_DETECT_MINB_LIGHT : DEM_DETECT_MINB) *
                                                      256 / DEM_DETECT_TPB) k_detect(StepBuffers b, DevGrid g,
                                                                 uint32_t N, uint32_t K, float S2c) {
  pdl_enter();
  const uint32_t err = ld_volatile(&b.err->code);  // checked once the first loads are out
  uint32_t jlo, jhi;
  owned_range(b, g, N, jlo, jhi);
  const uint32_t lane = lane_id();
  const uint32_t j = jlo + blockIdx.x * blockDim.x + threadIdx.x;
  if (j - lane >= jhi) return;  // whole warp past the end (warp-uniform)
  const bool valid = j < jhi;
  float4 P = valid ? __ldg(&b.pos_sorted[j]) : make_float4(0.f, 0.f, 0.f, 0.f);
  if (MONO) P.w = b.sw_r;
  if (err != 0u) return;  // warp-uniform
  uint32_t npair = 0;
  if (valid) {
    // own cell: the step-2 hash of the own position (identical to CM by construction)
    const int cx = cell_coord(P.x, g.lo[0], g.inv_h, g.nx);
    const int cy = cell_coord(P.y, g.lo[1], g.inv_h, g.ny);
    const int cz = cell_coord(P.z, g.lo[2], g.inv_h, g.nz_global) - g.zlo;
    float amb = -1.f;
    npair = detect_scan<false, MONO>(b, g, P, cx, cy, cz, j, b.clist + j, N, K, amb, S2c);
    if (amb >= 0.f)
      npair = detect_scan<true, MONO>(b, g, P, cx, cy, cz, j, b.clist + j, N, K, amb, S2c);
  }
  // the warp — the 32 sorted slots of one k_force warp — scans its (capped)
  // counts: each slot's first contact in the warp's flattened order, its
  // count and an overflow bit, so k_force needs no scan
  const uint32_t n = min(npair, K);
  uint32_t incl = n;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= (uint32_t)d) incl += v;
  }
  if (valid) __stcg(&b.ccount[j], (incl - n) | (n << 16) | (npair > K ? 0x80000000u : 0u));
}

// k_force: warp per 32 consecutive sorted particles. The warp's contacts are
// flattened and dealt round-robin to all 32 lanes, so a round evaluates 32
// contacts (Eqs. 2-10) regardless of which particles own them — the
// divergence of §6 (~12 contacts among ~47 candidates
// leaves 3/4 of a thread-per-particle warp idle) is removed from the
// expensive part. Each round's results go to shared memory and every owner
// adds its own contacts in candidate order (deterministic; the oracle's
// order). Partner slots are translated to old slots once per warp, so a round
// issues its partner-state and history loads together. δ_t,old is read at the
// contact's own list index first (persisting contacts keep their position).
// Two configurations of the same kernel, chosen per handle from the measured
// contacts per particle (dem_api.cu, choose_force_cfg); identical arithmetic
// and summation order, so their results are bitwise equal:
//   kForceDense (0): owner state in registers, broadcast by 12 shuffles per
//     round; partner old slots staged per (k, lane); 72 registers, 7 blocks/SM.
//     Best when a warp has many rounds (c̄ ≳ 8: C2, C3).
//   kForceLight (1): owner velocity and spin in shared memory (4 shuffles per
//     round for the position), partner old slots staged in chunks of 256
//     contacts; 64 registers, 8 blocks/SM. Best for c̄ ≲ 8 (C4, C5).
// Both keep each window of two rounds' results in shared memory and let the
// owners accumulate once per window.
constexpr int kForceDense = 0, kForceLight = 1;
// k_force blocks: DEM_SWEEP_WARPS warps each; resident warps per SM the
// register budget targets: light 32 (64 registers), dense 28 (72)
#ifndef DEM_SWEEP_WARPS
#define DEM_SWEEP_WARPS 1
#endif
#ifndef DEM_LIGHT_MINB
#define DEM_LIGHT_MINB (32 / DEM_SWEEP_WARPS)
#endif
#ifndef DEM_LIGHT_CHUNK
#define DEM_LIGHT_CHUNK 256u
#endif
template <int CFG>
struct ForceCfg {
  static constexpr bool kOwnSmem = CFG == kForceLight;
  static constexpr uint32_t kChunk = CFG == kForceLight ? DEM_LIGHT_CHUNK : 0u;  // 0: per (k, lane)
  static constexpr int kMinBlocks = CFG == kForceLight ? DEM_LIGHT_MINB : 28 / DEM_SWEEP_WARPS;
};
#ifndef DEM_RES_W
#define DEM_RES_W 64
#endif
constexpr uint32_t kResW = DEM_RES_W;  // contacts per accumulation window (two rounds)
struct WarpSmemLayout {
  uint32_t bytes, pf, cq, res, own, ost, base, slot, nold;
  // fixed-size regions first, so their offsets are compile-time constants;
  // the K-dependent ones (partner slots, owner map) last
  // fused (k_force<..., FUSED>): the warp's own detection fills the partner
  // list per (k, lane), as in the dense configuration
  __host__ __device__ static WarpSmemLayout make(uint32_t K, int cfg, bool fused = false) {
    WarpSmemLayout L;
    uint32_t o = 0;
    L.pf = o;
    o += 4 * 32 * 16;  // prefetch buffer: partner pos, vel, omg, predicted δ_t,old entry
    L.res = o;
    o += kResW * 24;  // results window: float4 (F_c, Tc.x), then float2 (Tc.y, Tc.z)
    L.ost = o;
    if (cfg == kForceLight) o += 2 * 32 * 16;  // owner V, W per lane
    L.base = o;
    o += 36 * 4;
    L.slot = o;
    o += 32 * 4;
    L.nold = o;
    o += 32 * 4;
    L.cq = o;
    o += (cfg == kForceLight && !fused ? ForceCfg<kForceLight>::kChunk : K * 32) * 4;  // partner old slots
    L.own = o;
    o += ((K * 32 + 15u) & ~15u);  // owner lane of each contact
    L.bytes = (o + 15u) & ~15u;
    return L;
  }
};
constexpr int kSweepWarps = DEM_SWEEP_WARPS;  // warps per k_force block
constexpr uint32_t kForceKC = 16;  // K with its own k_force instantiation
// K = 32 (the polydisperse C5) with its own light instantiation too
#ifndef DEM_FORCE_KC32
#define DEM_FORCE_KC32 1
#endif
#ifndef DEM_FORCE_FIRST
#define DEM_FORCE_FIRST 4
#endif
#ifndef DEM_HIST_UNCOND
#define DEM_HIST_UNCOND 1
#endif
constexpr int kForceFirst = DEM_FORCE_FIRST;  // list entries read before the count arrives
constexpr bool kHistUncond = DEM_HIST_UNCOND != 0;

// δ_t,old of partner `pid` in the old list of old slot s (n entries) when
// the caller's guess, index k (the contact's own index in the new list;
// n: none), missed (R10: absent -> 0). Lists are in candidate order, so a
// contact that formed or broke earlier in the list shifts the rest by one:
// entries k - 1 and k + 1 are tried first, then the others in order. (A scan
// from 0 cost a dependent L2 round trip per entry before the shifted entry,
// and ~1-3% of the C4 contacts miss their guess — a third to half of the
// 32-contact rounds.) Serial on purpose: a wider probe raised the register
// pressure of the common path (spills in k_force's round loop).
__device__ __forceinline__ f3 old_history(const float4* __restrict__ hist_in, uint32_t K,
                                          uint32_t s, uint32_t n, uint32_t k, uint32_t pid) {
  const float4* __restrict__ h = hist_in + (size_t)s * K;
  for (uint32_t t = 0; t < n + 2u; ++t) {
    const uint32_t x = t == 0u ? k - 1u : t == 1u ? k + 1u : t - 2u;
    if (x >= n || (t >= 2u && x + 1u - k <= 2u)) continue;  // out of range / tried already
    const float4 e = __ldcs(&h[x]);
    if (__float_as_uint(e.w) == pid) return mk(e.x, e.y, e.z);
  }
  return mk(0.f, 0.f, 0.f);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 16-byte global -> shared asynchronous copy (LDGSTS), L2 only (.cg; the
// L1-allocating .ca measured slower, profiles/r1_history.md #18).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src)
               : "memory");
}
// the same with the shared-memory destination as a 32-bit shared address
__device__ __forceinline__ void cp_async16_s(uint32_t smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gmem_src)
               : "memory");
}
// round-1 history #52, reproduced (DEM_HIST_HINT): the δ_t,old prefetch with
// an L2 evict-first policy. DEM_HIST_HINT=1 writes the policy where PTX also
// accepts the optional src-size operand — a 32-bit register there is taken
// as src-size (bytes copied, the rest of the 16 zero-filled): the defect that
// made a parity test fail in round 1; DEM_HIST_HINT=2 passes the 64-bit policy
// from createpolicy, which is the cache-policy operand.
#ifndef DEM_HIST_HINT
#define DEM_HIST_HINT 0
#endif
__device__ __forceinline__ void cp_async16_hist(uint32_t smem_dst, const void* gmem_src) {
#if DEM_HIST_HINT == 1
  uint32_t pol32;
  asm volatile("{.reg .b64 p; createpolicy.fractional.L2::evict_first.b64 p, 1.0; cvt.u32.u64 %0, p;}"
               : "=r"(pol32));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(gmem_src),
               "r"(pol32)
               : "memory");
#elif DEM_HIST_HINT == 2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_dst),
               "l"(gmem_src), "l"(pol)
               : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gmem_src)
               : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N_PENDING>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N_PENDING) : "memory");
}

// KC: the list capacity K as a compile-time constant (0: the runtime Kr), so
// the shared-memory layout and the history addressing fold to constants.
// FUSED (one radius only, b.sw_r > 0): the warp detects its own contacts
// first (steps 5-6, the scan of k_detect into its shared-memory list) — no
// k_detect launch, no contact list or (base, n) words in HBM.
// With the detection fused in, both configurations take 28 blocks per SM (72
// registers): the light one measured 2% faster than at 32 (r2 history #32)
#ifndef DEM_FUSED_MINB
#define DEM_FUSED_MINB (28 / DEM_SWEEP_WARPS)
#endif
template <int MODEL, bool DIAG, int CFG, bool MAT, uint32_t KC = 0, bool FUSED = false>
__global__ void __launch_bounds__(32 * kSweepWarps, FUSED ? DEM_FUSED_MINB : ForceCfg<CFG>::kMinBlocks)
    k_force(StepBuffers b, DevGrid g, DevPhys ph, uint32_t N, uint32_t Kr) {
  using C = ForceCfg<CFG>;
  constexpr uint32_t kChunk = FUSED ? 0u : C::kChunk;  // 0: partner slots per (k, lane)
  const uint32_t K = KC ? KC : Kr;
  pdl_enter();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t err = ld_volatile(&b.err->code);  // checked once the first loads are out
  const WarpSmemLayout L = WarpSmemLayout::make(K, CFG, FUSED);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint8_t* ws = smem_raw + (size_t)warp * L.bytes;
  float4* pf = reinterpret_cast<float4*>(ws + L.pf);                 // [field][lane]
  uint32_t* s_cq = reinterpret_cast<uint32_t*>(ws + L.cq);           // partner old slots
  float4* s_r4 = reinterpret_cast<float4*>(ws + L.res);              // [m % kResW]: F_c, Tc.x
  float2* s_r2 = reinterpret_cast<float2*>(ws + L.res + kResW * 16);  // [m % kResW]: Tc.y, Tc.z
  uint8_t* s_own = ws + L.own;                                       // owner of each contact
  float4* s_ost = reinterpret_cast<float4*>(ws + L.ost);             // light: [V | W][lane]
  uint32_t* s_base = reinterpret_cast<uint32_t*>(ws + L.base);       // [33]
  uint32_t* s_slot = reinterpret_cast<uint32_t*>(ws + L.slot);
  uint32_t* s_nold = reinterpret_cast<uint32_t*>(ws + L.nold);

  uint32_t jlo, jhi;
  owned_range(b, g, N, jlo, jhi);
  const uint32_t j0 = jlo + (blockIdx.x * kSweepWarps + warp) * 32u;
  const uint32_t j = j0 + lane;
  const bool valid = j < jhi;
  if (j0 >= jhi) return;  // whole warp past the end

  // ---- own particle (step 4 gather through SCCM) and its contact list. The
  // first four list entries are read before the count is known (entries past
  // the count are never used), so they do not wait for it.
  // one radius (b.sw_r > 0): the sorted position carries the old slot SCCM[j]
  // in .w and the lists hold partner old slots, so no SCCM gathers at all
  const bool sw = FUSED || b.sw_r > 0.f;
  Own o;
  o.P = valid ? __ldg(&b.pos_sorted[j]) : make_float4(0.f, 0.f, 0.f, 1.f);
  const uint32_t meta = valid && !FUSED ? __ldcs(&b.ccount[j]) : 0u;  // k_detect's (base, n) word
  uint32_t t_first[kForceFirst];
#pragma unroll
  for (int u = 0; u < kForceFirst; ++u)
    t_first[u] = valid && !FUSED && u < K ? __ldcs(&b.clist[(size_t)u * N + j]) : 0u;
  const uint32_t s = !valid ? 0u : sw ? __float_as_uint(o.P.w) : __ldcs(&b.perm[j]);
  if (sw) o.P.w = valid ? b.sw_r : 1.f;
  if (err != 0u) return;  // warp-uniform (one load per warp instruction)
  o.V = valid ? __ldg(&b.vel_in[s]) : make_float4(0.f, 0.f, 0.f, 1.f);
  o.W = valid ? __ldg(&b.omg_in[s]) : make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t n_old = (MODEL == 0 && valid) ? min(__ldcs(&b.cnt_in[s]), K) : 0u;
  bool overflow;
  uint32_t npair, mybase, M;
  uint32_t sk = 0xFFFFFFFFu;  // this step's key of the own position (fused: from the detection)
  if (FUSED) {
    // steps 5-6 for the warp's 32 slots (k_detect's scan, the list kept in
    // shared memory) while the owner state loads above are in flight
    uint32_t np = 0;
    if (valid) {
      const int cx = cell_coord(o.P.x, g.lo[0], g.inv_h, g.nx);
      const int cy = cell_coord(o.P.y, g.lo[1], g.inv_h, g.ny);
      const int cz = cell_coord(o.P.z, g.lo[2], g.inv_h, g.nz_global) - g.zlo;
      sk = (uint32_t)cx + (uint32_t)g.nx * ((uint32_t)cy + (uint32_t)g.ny * (uint32_t)cz);
      const float S = b.sw_r + b.sw_r, S2c = S * S;
      float amb = -1.f;
      np = detect_scan<false, true, true, CFG == kForceDense,
                       CFG == kForceDense ? kDetectFlatDense : kDetectFlat>(
          b, g, o.P, cx, cy, cz, j, s_cq + lane, 32u, K, amb, S2c);
      if (amb >= 0.f)  // a candidate in the ±16u band: the exact rescan (R14)
        np = detect_scan<true, true, true>(b, g, o.P, cx, cy, cz, j, s_cq + lane, 32u, K, amb, S2c);
    }
    overflow = np > K;
    npair = min(np, K);
    uint32_t incl = npair;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= (uint32_t)d) incl += v;
    }
    mybase = incl - npair;
    M = __shfl_sync(0xffffffffu, incl, 31);
  } else {
    overflow = (meta >> 31) != 0u;
    npair = (meta >> 16) & 0xFFu;
    mybase = meta & 0xFFFFu;
    M = __reduce_max_sync(0xffffffffu, mybase + npair);
  }
  s_slot[lane] = s;
  s_nold[lane] = n_old;
  if (C::kOwnSmem) {
    s_ost[lane] = o.V;
    s_ost[32 + lane] = o.W;
  }
  s_base[lane] = mybase;
  if (lane == 31) s_base[32] = M;
  for (uint32_t k = 0; k < npair; ++k) s_own[mybase + k] = (uint8_t)lane;
  // partner sorted slots -> old slots (SCCM), four lookups in flight per lane:
  // dense, all of them into s_cq[k*32 + lane]; light, those of the warp's
  // contacts [c0, c0 + kChunk) into s_cq[m - c0]
  auto translate = [&](uint32_t c0) {
    const uint32_t klo = kChunk ? (c0 > mybase ? c0 - mybase : 0u) : 0u;
    const uint32_t khi = kChunk ? min(npair, c0 + kChunk > mybase ? c0 + kChunk - mybase : 0u)
                                : npair;
    for (uint32_t k0 = klo; k0 < khi; k0 += 4) {
      uint32_t t4[4], q4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        t4[u] = k0 == 0                       ? t_first[u]
                : kForceFirst > 4 && k0 == 4 ? t_first[(kForceFirst > 4 ? 4 : 0) + u]
                        : (k0 + u < khi ? __ldcs(&b.clist[(size_t)(k0 + u) * N + j]) : 0u);
#pragma unroll
      for (int u = 0; u < 4; ++u) q4[u] = k0 + u < khi ? (sw ? t4[u] : __ldg(&b.perm[t4[u]])) : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u < khi) s_cq[kChunk ? mybase + k0 + u - c0 : (k0 + u) * 32 + lane] = q4[u];
    }
  };
  if (!FUSED) translate(0);  // (fused: the detection wrote the old slots already)
  __syncwarp();

  // prefetch of round r0's partner state + predicted δ_t,old entry (the
  // contact's own index in the owner's old list) into the buffer
  const uint32_t pf_s = smem_u32(pf) + lane * 16u;  // this lane's prefetch slots (shared addr)
  auto prefetch = [&](uint32_t r0) {
    const uint32_t m = r0 + lane;
    if (m < M) {
      const uint32_t ow = s_own[m];
      const uint32_t k = m - s_base[ow];
      const uint32_t q = kChunk ? s_cq[m % kChunk] : s_cq[k * 32 + ow];
      cp_async16_s(pf_s, &b.pos_in[q]);
      cp_async16_s(pf_s + 32u * 16u, &b.vel_in[q]);
      if (MODEL == 0) {
        cp_async16_s(pf_s + 64u * 16u, &b.omg_in[q]);
        // (unconditional: k < K is in bounds and the use checks k < n_old, so
        // the copy does not wait for the owner's history count)
        if (kHistUncond || k < s_nold[ow]) cp_async16_hist(pf_s + 96u * 16u, &b.hist_in[hix(s_slot[ow], k, K)]);
      }
    }
    cp_async_commit();
  };

  // ---- the warp's M contacts, 32 per round (step 7), next round in flight
  f3 F = mk(0.f, 0.f, 0.f), T = mk(0.f, 0.f, 0.f);
  if (M > 0) prefetch(0);
  for (uint32_t r0 = 0; r0 < M; r0 += 32) {
    cp_async_wait<0>();
    const float4 Q = pf[lane], VQ = pf[32 + lane], WQ = pf[64 + lane], Hr = pf[96 + lane];
    if (r0 + 32 < M) {
      __syncwarp();
      if (kChunk && (r0 + 32) % kChunk == 0) {  // the next round opens a new chunk
        translate(r0 + 32);
        __syncwarp();
      }
      prefetch(r0 + 32);  // overwrite the buffer: this round's data is in registers
    }
    const uint32_t m = r0 + lane;
    const uint32_t ow = m < M ? s_own[m] : 0u;
    // owner state: position from the owner lane's registers (all lanes take
    // part), velocity and spin likewise (dense) or from shared memory (light)
    Own po;
    po.P.x = __shfl_sync(0xffffffffu, o.P.x, ow);
    po.P.y = __shfl_sync(0xffffffffu, o.P.y, ow);
    po.P.z = __shfl_sync(0xffffffffu, o.P.z, ow);
    po.P.w = __shfl_sync(0xffffffffu, o.P.w, ow);
    if (C::kOwnSmem) {
      po.V = s_ost[ow];
      po.W = s_ost[32 + ow];
    } else {
      po.V.x = __shfl_sync(0xffffffffu, o.V.x, ow);
      po.V.y = __shfl_sync(0xffffffffu, o.V.y, ow);
      po.V.z = __shfl_sync(0xffffffffu, o.V.z, ow);
      po.V.w = __shfl_sync(0xffffffffu, o.V.w, ow);
      po.W.x = __shfl_sync(0xffffffffu, o.W.x, ow);
      po.W.y = __shfl_sync(0xffffffffu, o.W.y, ow);
      po.W.z = __shfl_sync(0xffffffffu, o.W.z, ow);
      po.W.w = __shfl_sync(0xffffffffu, o.W.w, ow);
    }
    f3 Fc = mk(0.f, 0.f, 0.f), Tc = mk(0.f, 0.f, 0.f);
    if (m < M) {
      const uint32_t k = m - s_base[ow];
      f3 n;
      float delta;
      if (!contact_geometry(po.P, Q, n, delta)) {
        raise_error(b.err, 9u, j0 - jlo + ow, __float_as_uint(po.W.w) & (MAT ? ph.idmask : 0xFFFFFFFFu));
      } else if (MODEL == 0) {
        const uint32_t pid = __float_as_uint(WQ.w) & (MAT ? ph.idmask : 0xFFFFFFFFu);
        const uint32_t no = s_nold[ow];
        f3 dold;
        if (k < no && __float_as_uint(Hr.w) == pid)
          dold = mk(Hr.x, Hr.y, Hr.z);
        else
          dold = old_history(b.hist_in, K, s_slot[ow], no, k, pid);
        f3 dnew;
        eval_pair_practical<MAT>(po, Q, VQ, WQ, n, delta, dold, ph, Fc, Tc, dnew);
        __stcs(&b.hist_out[hix((j0 - jlo) + ow, k, K)],
               make_float4(dnew.x, dnew.y, dnew.z, __uint_as_float(pid)));
      } else {
        const f3 u = mk(VQ.x - po.V.x, VQ.y - po.V.y, VQ.z - po.V.z);
        Fc = pair_simple(n, delta, u, ph.ksp, ph.kda, ph.ksh);
      }
    }
    const uint32_t w0 = r0 - r0 % kResW;  // first contact of the current window
    s_r4[r0 - w0 + lane] = make_float4(Fc.x, Fc.y, Fc.z, Tc.x);
    if (MODEL == 0) s_r2[r0 - w0 + lane] = make_float2(Tc.y, Tc.z);
    if (r0 + 32 - w0 == kResW || r0 + 32 >= M) {  // window full (or last round)
      __syncwarp();
      // each owner adds its contacts of this window, in candidate order
      const uint32_t lo = max(mybase, w0), hi = min(mybase + npair, r0 + 32);
#pragma unroll 4
      for (uint32_t x = lo; x < hi; ++x) {
        const float4 r4 = s_r4[x - w0];
        F = mk(F.x + r4.x, F.y + r4.y, F.z + r4.z);
        if (MODEL == 0) {
          const float2 r2 = s_r2[x - w0];
          T = mk(T.x + r4.w, T.y + r2.x, T.z + r2.y);
        }
      }
      __syncwarp();
    }
  }
  if (!valid) return;
  if (C::kOwnSmem) {  // (those registers were free during the rounds)
    o.V = s_ost[lane];
    o.W = s_ost[32 + lane];
  }
  if (MODEL == 0) T = mk(o.P.w * T.x, o.P.w * T.y, o.P.w * T.z);  // Eq. 3: r_i Σ n × F_t
  auto lookup = [&](uint32_t pid) -> f3 {  // walls: after the pair contacts in the old list
    return old_history(b.hist_in, K, s, n_old, n_old, pid);
  };
  finish_particle<MODEL, DIAG, MAT>(b, g, ph, N, K, j - jlo, o, F, T, npair, overflow, lookup, sk);
}

#if DEM_ABLATIONS  // (libdem_ablations.so only)
// ---- ablation: warp-specialised k_force (DEM_F_FORCE_WS) ------------------
// The same step as k_force, split by role. A block holds 4 producer warps
// (warpgroup 0, registers cut to 40 by setmaxnreg) and 4 consumer warps
// (warpgroup 1, raised to 88), paired one to one; each pair walks its
// 32-slot groups (persistent: one wave of blocks, groups strided). The
// producer does everything that waits on memory: the group's entry data
// (sorted position, (base, n) word, list entries, owner state through the
// old slot, the old history count), the owner map and the slot
// translation, and per round the partner state and predicted δ_t,old entry
// (cp.async) plus each contact's (owner lane, list index) — into a ring of
// shared-memory slots, a group header first, then its rounds. The consumer
// only computes: owner state from the header into registers (broadcast by
// shuffles), the contact arithmetic (Eqs. 2-10), the owners' accumulation
// in candidate order, the walls, the integration and the stores. Ring slots
// are handed over by mbarriers: "full" completes when the producer's
// copies have landed (cp.async.mbarrier.arrive.noinc) and its plain stores
// are released (mbarrier.arrive), "empty" when the consumer has read the
// slot. Same arithmetic and summation order as k_force: bitwise-identical
// results.
#ifndef DEM_WS_SLEEP
#define DEM_WS_SLEEP 200  // ns the producer sleeps between polls of a busy slot
#endif
#ifndef DEM_WS_SLOTS
#define DEM_WS_SLOTS 3
#endif
#ifndef DEM_WS_BLOCKS  // blocks per SM; producer / consumer registers follow
#define DEM_WS_BLOCKS 4
#endif
#ifndef DEM_WS_PREG
#define DEM_WS_PREG 40
#endif
#ifndef DEM_WS_CREG
#define DEM_WS_CREG 88
#endif
constexpr int kWsPairs = 4;  // producer/consumer warp pairs per block
constexpr int kWsSlots = DEM_WS_SLOTS;  // ring slots per pair
struct WsSlot {
  float4 f[4][32];    // round: partner pos, vel, omg, δ_t,old entry; header: P, V, W, (meta, s, nold)
  uint32_t meta[32];  // round: owner lane | list index << 8 (0xFFFFFFFF: no contact)
};
struct WsLayout {  // per pair, inside the block's dynamic shared memory
  uint32_t slots, bars, own, cq, res, bytes;
  __host__ __device__ static WsLayout make(uint32_t K) {
    WsLayout L;
    uint32_t o = 0;
    L.slots = o;
    o += kWsSlots * (uint32_t)sizeof(WsSlot);
    L.bars = o;
    o += 2 * kWsSlots * 8;  // full[], empty[] mbarriers
    L.own = o;
    o += (K * 32 + 15u) & ~15u;  // producer: owner lane of each contact
    L.cq = o;
    o += K * 32 * 4;  // producer: partner old slots [k][lane]
    L.res = o;
    o += kResW * 24;  // consumer: results window
    L.bytes = (o + 15u) & ~15u;
    return L;
  }
};

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{.reg .b64 st; mbarrier.arrive.shared.b64 st, [%0];}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
// the producer's wait for a free slot backs off, so its spinning does not take
// issue slots from the consumers (it is ahead by construction)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  for (;;) {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    if (ok) return;
    __nanosleep(DEM_WS_SLEEP);
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{.reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

template <int MODEL, bool DIAG, bool MAT, uint32_t KC = 0>
__global__ void __launch_bounds__(32 * 2 * kWsPairs, DEM_WS_BLOCKS)
    k_force_ws(StepBuffers b, DevGrid g, DevPhys ph, uint32_t N, uint32_t Kr) {
  const uint32_t K = KC ? KC : Kr;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t err = ld_volatile(&b.err->code);
  const WsLayout L = WsLayout::make(K);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const bool producer = warp < (uint32_t)kWsPairs;
  const uint32_t pair = producer ? warp : warp - kWsPairs;
  uint8_t* ps = smem_raw + (size_t)pair * L.bytes;
  WsSlot* slots = reinterpret_cast<WsSlot*>(ps + L.slots);
  uint64_t* full = reinterpret_cast<uint64_t*>(ps + L.bars);
  uint64_t* empty = full + kWsSlots;
  if (producer && lane == 0) {
    for (int i = 0; i < kWsSlots; ++i) {
      mbar_init(&full[i], 64);   // 32 async (copies landed) + 32 plain arrivals
      mbar_init(&empty[i], 32);  // the consumer's lanes
    }
  }
  __syncthreads();
  if (err != 0u) return;  // (block-uniform: before any barrier use)
  uint32_t jlo, jhi;
  owned_range(b, g, N, jlo, jhi);
  const uint32_t ngroups = (jhi - jlo + 31u) >> 5;
  const uint32_t stride = gridDim.x * kWsPairs;
  const bool sw = b.sw_r > 0.f;
  uint32_t use = 0;  // ring uses so far (slot = use % kWsSlots, its phase = use / kWsSlots)

  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(DEM_WS_PREG));
    uint8_t* s_own = ps + L.own;
    uint32_t* s_cq = reinterpret_cast<uint32_t*>(ps + L.cq);
    auto acquire = [&]() -> WsSlot* {
      const uint32_t i = use % kWsSlots;
      if (use >= (uint32_t)kWsSlots) mbar_wait_backoff(&empty[i], ((use / kWsSlots) - 1u) & 1u);
      return &slots[i];
    };
    auto publish = [&]() {
      uint64_t* f = &full[use % kWsSlots];
      mbar_arrive_cp_async(f);
      mbar_arrive(f);
      ++use;
    };
    for (uint32_t grp = blockIdx.x * kWsPairs + pair; grp < ngroups; grp += stride) {
      const uint32_t j0 = jlo + grp * 32u, j = j0 + lane;
      const bool valid = j < jhi;
      float4 P = valid ? __ldg(&b.pos_sorted[j]) : make_float4(0.f, 0.f, 0.f, 1.f);
      const uint32_t meta = valid ? __ldcs(&b.ccount[j]) : 0u;
      uint32_t t_first[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t_first[u] = valid && (uint32_t)u < K ? __ldcs(&b.clist[(size_t)u * N + j]) : 0u;
      const uint32_t s = !valid ? 0u : sw ? __float_as_uint(P.w) : __ldcs(&b.perm[j]);
      if (sw) P.w = valid ? b.sw_r : 1.f;
      const uint32_t npair = (meta >> 16) & 0xFFu, mybase = meta & 0xFFFFu;
      const uint32_t M = __reduce_max_sync(0xffffffffu, mybase + npair);
      const uint32_t n_old = (MODEL == 0 && valid) ? min(__ldcs(&b.cnt_in[s]), K) : 0u;
      // the group header: owner position, velocity, spin, (base/n word, old slot, count)
      WsSlot* hs = acquire();
      hs->f[0][lane] = P;
      if (valid) {
        cp_async16(&hs->f[1][lane], &b.vel_in[s]);
        cp_async16(&hs->f[2][lane], &b.omg_in[s]);
      } else {
        hs->f[1][lane] = make_float4(0.f, 0.f, 0.f, 1.f);
        hs->f[2][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      reinterpret_cast<uint4*>(&hs->f[3][0])[lane] = make_uint4(meta, s, n_old, 0u);
      cp_async_commit();
      publish();
      // owner map and partner old slots (round 1's scheme, in the producer)
      for (uint32_t k = 0; k < npair; ++k) s_own[mybase + k] = (uint8_t)lane;
      for (uint32_t k0 = 0; k0 < npair; k0 += 4) {
        uint32_t t4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          t4[u] = k0 == 0 ? t_first[u]
                          : (k0 + u < npair ? __ldcs(&b.clist[(size_t)(k0 + u) * N + j]) : 0u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k0 + u < npair) s_cq[(k0 + u) * 32u + lane] = sw ? t4[u] : __ldg(&b.perm[t4[u]]);
      }
      __syncwarp();
      for (uint32_t r0 = 0; r0 < M; r0 += 32) {
        const uint32_t m = r0 + lane;
        const uint32_t ow = m < M ? s_own[m] : 0u;
        const uint32_t bo = __shfl_sync(0xffffffffu, mybase, ow);
        const uint32_t so = __shfl_sync(0xffffffffu, s, ow);
        WsSlot* rs = acquire();
        if (m < M) {
          const uint32_t k = m - bo;
          const uint32_t q = s_cq[k * 32u + ow];
          cp_async16(&rs->f[0][lane], &b.pos_in[q]);
          cp_async16(&rs->f[1][lane], &b.vel_in[q]);
          if (MODEL == 0) {
            cp_async16(&rs->f[2][lane], &b.omg_in[q]);
            cp_async16(&rs->f[3][lane], &b.hist_in[hix(so, k, K)]);  // (k < K: in bounds)
          }
          rs->meta[lane] = ow | (k << 8);
        } else {
          rs->meta[lane] = 0xFFFFFFFFu;
        }
        cp_async_commit();
        publish();
      }
      __syncwarp();  // (s_own / s_cq of this group read by all lanes before the next group)
    }
    return;
  }

  // ---------------------------------------------------------------- consumer
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(DEM_WS_CREG));
  float4* s_r4 = reinterpret_cast<float4*>(ps + L.res);
  float2* s_r2 = reinterpret_cast<float2*>(ps + L.res + kResW * 16);
  auto take = [&]() -> const WsSlot* {
    const uint32_t i = use % kWsSlots;
    mbar_wait(&full[i], (use / kWsSlots) & 1u);
    return &slots[i];
  };
  auto give = [&]() {
    mbar_arrive(&empty[use % kWsSlots]);
    ++use;
  };
  for (uint32_t grp = blockIdx.x * kWsPairs + pair; grp < ngroups; grp += stride) {
    const uint32_t j0 = jlo + grp * 32u, j = j0 + lane;
    const bool valid = j < jhi;
    const WsSlot* hs = take();
    Own o;
    o.P = hs->f[0][lane];
    o.V = hs->f[1][lane];
    o.W = hs->f[2][lane];
    const uint4 hm = reinterpret_cast<const uint4*>(&hs->f[3][0])[lane];
    give();
    const uint32_t meta = hm.x, s = hm.y, n_old = hm.z;
    const bool overflow = (meta >> 31) != 0u;
    const uint32_t npair = (meta >> 16) & 0xFFu, mybase = meta & 0xFFFFu;
    const uint32_t M = __reduce_max_sync(0xffffffffu, mybase + npair);
    f3 F = mk(0.f, 0.f, 0.f), T = mk(0.f, 0.f, 0.f);
    for (uint32_t r0 = 0; r0 < M; r0 += 32) {
      const WsSlot* rs = take();
      const float4 Q = rs->f[0][lane], VQ = rs->f[1][lane];
      const float4 WQ = MODEL == 0 ? rs->f[2][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 Hr = MODEL == 0 ? rs->f[3][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t cm = rs->meta[lane];
      give();
      const uint32_t m = r0 + lane;
      const uint32_t ow = m < M ? (cm & 0xFFu) : 0u;
      const uint32_t k = cm >> 8;
      Own po;
      po.P.x = __shfl_sync(0xffffffffu, o.P.x, ow);
      po.P.y = __shfl_sync(0xffffffffu, o.P.y, ow);
      po.P.z = __shfl_sync(0xffffffffu, o.P.z, ow);
      po.P.w = __shfl_sync(0xffffffffu, o.P.w, ow);
      po.V.x = __shfl_sync(0xffffffffu, o.V.x, ow);
      po.V.y = __shfl_sync(0xffffffffu, o.V.y, ow);
      po.V.z = __shfl_sync(0xffffffffu, o.V.z, ow);
      po.V.w = __shfl_sync(0xffffffffu, o.V.w, ow);
      po.W.x = __shfl_sync(0xffffffffu, o.W.x, ow);
      po.W.y = __shfl_sync(0xffffffffu, o.W.y, ow);
      po.W.z = __shfl_sync(0xffffffffu, o.W.z, ow);
      po.W.w = __shfl_sync(0xffffffffu, o.W.w, ow);
      const uint32_t so = __shfl_sync(0xffffffffu, s, ow);
      const uint32_t no = __shfl_sync(0xffffffffu, n_old, ow);
      f3 Fc = mk(0.f, 0.f, 0.f), Tc = mk(0.f, 0.f, 0.f);
      if (m < M) {
        f3 n;
        float delta;
        if (!contact_geometry(po.P, Q, n, delta)) {
          raise_error(b.err, 9u, j0 - jlo + ow, __float_as_uint(po.W.w) & (MAT ? ph.idmask : 0xFFFFFFFFu));
        } else if (MODEL == 0) {
          const uint32_t pid = __float_as_uint(WQ.w) & (MAT ? ph.idmask : 0xFFFFFFFFu);
          f3 dold;
          if (k < no && __float_as_uint(Hr.w) == pid)
            dold = mk(Hr.x, Hr.y, Hr.z);
          else
            dold = old_history(b.hist_in, K, so, no, k, pid);
          f3 dnew;
          eval_pair_practical<MAT>(po, Q, VQ, WQ, n, delta, dold, ph, Fc, Tc, dnew);
          __stcs(&b.hist_out[hix((j0 - jlo) + ow, k, K)],
                 make_float4(dnew.x, dnew.y, dnew.z, __uint_as_float(pid)));
        } else {
          const f3 u = mk(VQ.x - po.V.x, VQ.y - po.V.y, VQ.z - po.V.z);
          Fc = pair_simple(n, delta, u, ph.ksp, ph.kda, ph.ksh);
        }
      }
      const uint32_t w0 = r0 - r0 % kResW;
      s_r4[r0 - w0 + lane] = make_float4(Fc.x, Fc.y, Fc.z, Tc.x);
      if (MODEL == 0) s_r2[r0 - w0 + lane] = make_float2(Tc.y, Tc.z);
      if (r0 + 32 - w0 == kResW || r0 + 32 >= M) {
        __syncwarp();
        const uint32_t lo = max(mybase, w0), hi = min(mybase + npair, r0 + 32);
#pragma unroll 4
        for (uint32_t x = lo; x < hi; ++x) {
          const float4 r4 = s_r4[x - w0];
          F = mk(F.x + r4.x, F.y + r4.y, F.z + r4.z);
          if (MODEL == 0) {
            const float2 r2 = s_r2[x - w0];
            T = mk(T.x + r4.w, T.y + r2.x, T.z + r2.y);
          }
        }
        __syncwarp();
      }
    }
    if (valid) {
      if (MODEL == 0) T = mk(o.P.w * T.x, o.P.w * T.y, o.P.w * T.z);  // Eq. 3: r_i Σ n × F_t
      auto lookup = [&](uint32_t pid) -> f3 {
        return old_history(b.hist_in, K, s, n_old, n_old, pid);
      };
      finish_particle<MODEL, DIAG, MAT>(b, g, ph, N, K, j - jlo, o, F, T, npair, overflow, lookup);
    }
  }
}

#endif  // DEM_ABLATIONS

#if DEM_ABLATIONS  // (libdem_ablations.so only)
// k_force_lane (configuration "lanes"): one thread per sorted particle walks
// its own compacted contact list (k_detect's, so §6's divergence of contacts
// among candidates stays out of it; what remains is the spread of list
// lengths inside a warp: 0.93 of the lanes busy on C4, 0.95 on C3, bench
// `analysis`). The owner's state stays in its registers — no shuffles, no
// owner map, no results window — and contact k+1's partner state and
// predicted δ_t,old entry are in flight (cp.async, double-buffered per
// thread) while contact k is evaluated; the list entry two ahead is loaded
// one contact earlier still. Same arithmetic and the same per-owner order
// as k_force, so the results are bitwise equal to the other configurations.
#ifndef DEM_LANES_MINB
#define DEM_LANES_MINB 8
#endif
constexpr int kLanesThreads = 128;
template <int MODEL, bool DIAG, bool MAT, uint32_t KC = 0>
__global__ void __launch_bounds__(kLanesThreads, DEM_LANES_MINB)
    k_force_lane(StepBuffers b, DevGrid g, DevPhys ph, uint32_t N, uint32_t Kr) {
  const uint32_t K = KC ? KC : Kr;
  pdl_enter();
  __shared__ float4 pf[2][4][kLanesThreads];  // [buffer][pos, vel, omg, hist][thread]
  const uint32_t err = ld_volatile(&b.err->code);  // checked once the first loads are out
  uint32_t jlo, jhi;
  owned_range(b, g, N, jlo, jhi);
  const uint32_t tid = threadIdx.x;
  const uint32_t j = jlo + blockIdx.x * kLanesThreads + tid;
  if (j >= jhi) return;  // (no block-level synchronisation below)
  const bool sw = b.sw_r > 0.f;
  Own o;
  o.P = __ldg(&b.pos_sorted[j]);
  const uint32_t meta = __ldcs(&b.ccount[j]);  // k_detect's (base, n) word
  // the first two list entries, before the count arrives (entries past the
  // count are never used)
  const uint32_t e0 = K > 0 ? __ldcs(&b.clist[j]) : 0u;
  const uint32_t e1 = K > 1 ? __ldcs(&b.clist[(size_t)N + j]) : 0u;
  const uint32_t s = sw ? __float_as_uint(o.P.w) : __ldcs(&b.perm[j]);
  if (sw) o.P.w = b.sw_r;
  if (err != 0u) return;
  const bool overflow = (meta >> 31) != 0u;
  const uint32_t npair = (meta >> 16) & 0xFFu;
  o.V = __ldg(&b.vel_in[s]);
  o.W = __ldg(&b.omg_in[s]);
  const uint32_t n_old = MODEL == 0 ? min(__ldcs(&b.cnt_in[s]), K) : 0u;
  // contact k's partner (list entry e) and history entry (s, k) -> buffer k & 1
  auto issue = [&](uint32_t k, uint32_t e) {
    const uint32_t q = sw ? e : __ldg(&b.perm[e]);
    float4(*buf)[kLanesThreads] = pf[k & 1u];
    cp_async16(&buf[0][tid], &b.pos_in[q]);
    cp_async16(&buf[1][tid], &b.vel_in[q]);
    if (MODEL == 0) {
      cp_async16(&buf[2][tid], &b.omg_in[q]);
      cp_async16(&buf[3][tid], &b.hist_in[hix(s, k, K)]);  // (k < K: in bounds; checked at use)
    }
    cp_async_commit();
  };
  // one contact in flight ahead of the one being evaluated (two ahead
  // measured no faster)
  if (npair > 0) issue(0, e0);
  uint32_t en = e1;                                                      // entry of contact k + 1
  uint32_t enn = npair > 2 ? __ldcs(&b.clist[(size_t)2 * N + j]) : 0u;  // of contact k + 2
  f3 F = mk(0.f, 0.f, 0.f), T = mk(0.f, 0.f, 0.f);
  for (uint32_t k = 0; k < npair; ++k) {
    if (k + 1 < npair) {
      issue(k + 1, en);
      en = enn;
      if (k + 3 < npair) enn = __ldcs(&b.clist[(size_t)(k + 3) * N + j]);
      cp_async_wait<1>();  // contact k's group is complete
    } else {
      cp_async_wait<0>();
    }
    const float4(*buf)[kLanesThreads] = pf[k & 1u];
    const float4 Q = buf[0][tid], VQ = buf[1][tid];
    f3 n;
    float delta;
    if (!contact_geometry(o.P, Q, n, delta)) {
      raise_error(b.err, 9u, j - jlo, __float_as_uint(o.W.w) & (MAT ? ph.idmask : 0xFFFFFFFFu));
    } else if (MODEL == 0) {
      const float4 WQ = buf[2][tid], Hr = buf[3][tid];
      const uint32_t pid = __float_as_uint(WQ.w) & (MAT ? ph.idmask : 0xFFFFFFFFu);
      const f3 dold = (k < n_old && __float_as_uint(Hr.w) == pid)
                          ? mk(Hr.x, Hr.y, Hr.z)
                          : old_history(b.hist_in, K, s, n_old, k, pid);
      f3 Fc, Tc, dnew;
      eval_pair_practical<MAT>(o, Q, VQ, WQ, n, delta, dold, ph, Fc, Tc, dnew);
      __stcs(&b.hist_out[hix(j - jlo, k, K)], make_float4(dnew.x, dnew.y, dnew.z, __uint_as_float(pid)));
      F = mk(F.x + Fc.x, F.y + Fc.y, F.z + Fc.z);
      T = mk(T.x + Tc.x, T.y + Tc.y, T.z + Tc.z);
    } else {
      const f3 u = mk(VQ.x - o.V.x, VQ.y - o.V.y, VQ.z - o.V.z);
      const f3 Fc = pair_simple(n, delta, u, ph.ksp, ph.kda, ph.ksh);
      F = mk(F.x + Fc.x, F.y + Fc.y, F.z + Fc.z);
    }
  }
  if (MODEL == 0) T = mk(o.P.w * T.x, o.P.w * T.y, o.P.w * T.z);  // Eq. 3: r_i Σ n × F_t
  auto lookup = [&](uint32_t pid) -> f3 {  // walls: after the pair contacts in the old list
    return old_history(b.hist_in, K, s, n_old, n_old, pid);
  };
  finish_particle<MODEL, DIAG, MAT>(b, g, ph, N, K, j - jlo, o, F, T, npair, overflow, lookup);
}

// ---- half-list ablation (DEM_F_HALF_LISTS): Newton's third law ----------
// Eq. 3/Eq. 4 with the R1 orientation make the pair force antisymmetric and
// the unscaled torque n x F_t symmetric, bitwise (P11): F_ji = -F_ij,
// δ_t,ji = -δ_t,ij, T_j = r_j Tc, T_i = r_i Tc. So each contact pair is
// evaluated once, by its lower sorted slot.
//   k_detect_half  candidates t > i (4.5 of the 9 rows; in slab mode also the
//                  low ghost rows), upper list of i, lower list of t (atomic
//                  append: t learns who evaluates its contacts)
//   k_pair         per upper contact: Eqs. 2-10, both history entries
//                  (δ_t on i's side, -δ_t on t's), the pair result R for t
//   k_finish       per particle: Σ over its lower contacts in ascending
//                  partner slot (deterministic) + its upper partial sum, walls,
//                  integration, next CM
// Each particle's history list is [upper | lower (append order) | walls];
// lookups are by partner id, so the order never changes a result.

__global__ void __launch_bounds__(256) k_detect_half(StepBuffers b, DevGrid g, uint32_t N,
                                                     uint32_t K) {
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t jlo = __ldg(&b.off[g.own_c0]), jhi = __ldg(&b.off[g.own_c1]);
  const uint32_t i = jlo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= jhi) return;
  const float4 P = __ldg(&b.pos_sorted[i]);
  const int cx = cell_coord(P.x, g.lo[0], g.inv_h, g.nx);
  const int cy = cell_coord(P.y, g.lo[1], g.inv_h, g.ny);
  const int cz = cell_coord(P.z, g.lo[2], g.inv_h, g.nz_global) - g.zlo;
  const uint32_t xa = cx > 0 ? (uint32_t)cx - 1u : 0u;
  const uint32_t xb = cx < g.nx - 1 ? (uint32_t)cx + 1u : (uint32_t)g.nx - 1u;
  const uint32_t nxy = (uint32_t)g.nx * (uint32_t)g.ny;
  uint32_t nup = 0;
  bool overflow = false;
#pragma unroll 1
  for (int dz = -1; dz <= 1; ++dz) {
    const int z = cz + dz;
    if (z < 0 || z >= g.nz) continue;
    uint32_t t0[3], t1[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int y = cy + r - 1;
      const bool in = y >= 0 && y < g.ny;
      const uint32_t row = (uint32_t)z * nxy + (uint32_t)(in ? y : 0) * (uint32_t)g.nx;
      t0[r] = in ? __ldg(&b.off[row + xa]) : 0u;
      t1[r] = in ? __ldg(&b.off[row + xb + 1]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      // this row's slots this particle evaluates: above i, or non-owned below jlo
      uint32_t lo = t0[r], hi = t1[r];
      if (lo <= i) lo = (hi > i) ? i + 1 : lo;  // the part above i
      const bool low_ghosts = t0[r] < jlo;     // rows of the low ghost plane (slab mode)
      if (!low_ghosts && lo >= hi) continue;
      if (!low_ghosts && t0[r] < i && t1[r] <= i) continue;  // row entirely below i
      const uint32_t ts = low_ghosts ? t0[r] : lo;
#pragma unroll 1
      for (uint32_t t = ts; t < hi; ++t) {
        if (t <= i && t >= jlo) continue;
        const float4 Q = __ldg(&b.pos_sorted[t]);
        const float dx = Q.x - P.x, dy = Q.y - P.y, dz2 = Q.z - P.z;
        const float d2 = dx * dx + dy * dy + dz2 * dz2;
        const float S = P.w + Q.w;
        const float S2 = S * S;
        bool hit = d2 <= S2 * 0.99999904632568359375f;  // (1 - 16u) S²: clearly touching
        if (!hit && d2 < S2 * 1.00000095367431640625f) {  // inside the band: exact (R14)
          const double Sd = (double)P.w + (double)Q.w;
          hit = exact_d2(P, Q) < __dmul_rn(Sd, Sd);
        }
        if (!hit) continue;
        if (nup >= K) {
          overflow = true;
          continue;
        }
        uint32_t p = 0xFFu;
        if (t >= jlo && t < jhi) {  // an owned partner learns who evaluates its contact
          p = atomicAdd(&b.lcount[t], 1u);
          if (p < K) __stcg(&b.llist[(size_t)p * N + t], (i << 5) | nup);
          else p = 0xFEu;  // partner overflow: raised by k_finish
        }
        __stcg(&b.clist[(size_t)nup * N + i], t);
        b.cpos[(size_t)nup * N + i] = (uint8_t)min(p, 0xFFu);
        ++nup;
      }
    }
  }
  __stcg(&b.ccount[i], overflow ? K + 1u : nup);
}

// k_pair: warp per 32 consecutive owned slots; the warp's upper contacts are
// flattened across its lanes (~2.6 per particle at C4, so ~3 full rounds).
// Each pair writes its result R (force on the lower particle, n x F_t) and
// both history entries; no accumulation here, so no owner bookkeeping beyond
// a shared-memory owner map.
template <int MODEL, bool MAT>
__global__ void __launch_bounds__(128) k_pair(StepBuffers b, DevGrid g, DevPhys ph, uint32_t N,
                                              uint32_t K) {
  __shared__ uint8_t s_own[4][32 * 32];
  __shared__ uint32_t s_base[4][33];
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t jlo = __ldg(&b.off[g.own_c0]), jhi = __ldg(&b.off[g.own_c1]);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t j0 = jlo + (blockIdx.x * 4u + warp) * 32u;
  if (j0 >= jhi) return;
  const uint32_t i_l = j0 + lane;
  const uint32_t nup = i_l < jhi ? min(__ldcs(&b.ccount[i_l]), K) : 0u;
  uint32_t incl = nup;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= (uint32_t)d) incl += v;
  }
  const uint32_t mybase = incl - nup;
  const uint32_t M = __shfl_sync(0xffffffffu, incl, 31);
  s_base[warp][lane] = mybase;
  for (uint32_t k = 0; k < nup; ++k) s_own[warp][mybase + k] = (uint8_t)lane;
  __syncwarp();
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t m = lane; m < M; m += 32) {
    const uint32_t ow = s_own[warp][m];
    const uint32_t k = m - s_base[warp][ow];
    const uint32_t i = j0 + ow;
    // first wave of independent loads
    const uint32_t t = __ldcs(&b.clist[(size_t)k * N + i]);
    const uint32_t cp = b.cpos[(size_t)k * N + i];
    const uint32_t si = __ldg(&b.perm[i]);
    Own o;
    o.P = __ldg(&b.pos_sorted[i]);
    const float4 Q = __ldg(&b.pos_sorted[t]);
    // second wave: through SCCM
    const uint32_t q = __ldg(&b.perm[t]);
    o.V = __ldg(&b.vel_in[si]);
    o.W = MODEL == 0 ? __ldg(&b.omg_in[si]) : z4;
    const uint32_t n_old = MODEL == 0 ? min(__ldcs(&b.cnt_in[si]), K) : 0u;
    const float4 Hk = (MODEL == 0 && k < K) ? __ldcs(&b.hist_in[hix(si, k, K)]) : z4;
    const uint32_t nup_t = (MODEL == 0 && cp < 0xFEu) ? min(__ldcs(&b.ccount[t]), K) : 0u;
    const float4 VQ = __ldg(&b.vel_in[q]);
    const float4 WQ = MODEL == 0 ? __ldg(&b.omg_in[q]) : z4;
    f3 n;
    float delta;
    f3 Fc = mk(0.f, 0.f, 0.f), Tc = mk(0.f, 0.f, 0.f);
    if (!contact_geometry(o.P, Q, n, delta)) {
      raise_error(b.err, 9u, i - jlo, __float_as_uint(o.W.w) & ph.idmask);
    } else if (MODEL == 0) {
      const uint32_t pid = __float_as_uint(WQ.w) & ph.idmask;
      const f3 dold = (k < n_old && __float_as_uint(Hk.w) == pid)
                          ? mk(Hk.x, Hk.y, Hk.z)
                          : old_history(b.hist_in, K, si, n_old, k, pid);
      f3 dnew;
      eval_pair_practical<MAT>(o, Q, VQ, WQ, n, delta, dold, ph, Fc, Tc, dnew);
      // this side's entry (upper part of i's list) and the partner's (lower part)
      __stcs(&b.hist_out[hix(i - jlo, k, K)],
             make_float4(dnew.x, dnew.y, dnew.z, __uint_as_float(pid)));
      if (cp < 0xFEu && nup_t + cp < K)
        __stcs(&b.hist_out[hix(t - jlo, nup_t + cp, K)],
               make_float4(-dnew.x, -dnew.y, -dnew.z,
                           __uint_as_float(__float_as_uint(o.W.w) & ph.idmask)));
    } else {
      const f3 u = mk(VQ.x - o.V.x, VQ.y - o.V.y, VQ.z - o.V.z);
      Fc = pair_simple(n, delta, u, ph.ksp, ph.kda, ph.ksh);
    }
    __stcs(&b.R0[(size_t)k * N + i], make_float4(Fc.x, Fc.y, Fc.z, Tc.x));
    if (MODEL == 0) __stcs(&b.R1[(size_t)k * N + i], make_float2(Tc.y, Tc.z));
  }
}

// k_finish: per particle, every contact's result in the oracle's order —
// lower partners ascending, then upper partners ascending (= ascending
// partner slot) — then walls and integration (finish_particle).
constexpr uint32_t kLowBatch = 8;  // lower-list entries sorted in registers
template <int MODEL, bool DIAG, bool MAT>
__global__ void __launch_bounds__(128) k_finish(StepBuffers b, DevGrid g, DevPhys ph, uint32_t N,
                                                uint32_t K) {
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t jlo = __ldg(&b.off[g.own_c0]), jhi = __ldg(&b.off[g.own_c1]);
  const uint32_t j = jlo + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= jhi) return;
  const uint32_t s = __ldcs(&b.perm[j]);
  const uint32_t nc = __ldcs(&b.ccount[j]);
  const uint32_t nlow_all = __ldcs(&b.lcount[j]);
  const uint32_t nlow = min(nlow_all, K);
  const uint32_t nup = min(nc, K);
  bool overflow = nc > K || nlow_all > K || nup + nlow > K;
  Own o;
  o.P = __ldg(&b.pos_sorted[j]);
  o.V = __ldg(&b.vel_in[s]);
  o.W = __ldg(&b.omg_in[s]);
  const uint32_t n_old = MODEL == 0 ? min(__ldcs(&b.cnt_in[s]), K) : 0u;
  f3 F = mk(0.f, 0.f, 0.f), T = mk(0.f, 0.f, 0.f);
  auto add = [&](float4 r0, float2 r1, float sign) {
    F = mk(F.x + sign * r0.x, F.y + sign * r0.y, F.z + sign * r0.z);
    if (MODEL == 0) T = mk(T.x + o.P.w * r0.w, T.y + o.P.w * r1.x, T.z + o.P.w * r1.y);
  };
  // lower contacts: entries (i << 5 | k) sort as the partner slot i
  uint32_t e[kLowBatch];
#pragma unroll
  for (uint32_t p = 0; p < kLowBatch; ++p)
    e[p] = p < nlow ? __ldcs(&b.llist[(size_t)p * N + j]) : 0xFFFFFFFFu;
#pragma unroll
  for (uint32_t a = 1; a < kLowBatch; ++a)  // insertion sort, fully unrolled (registers)
#pragma unroll
    for (uint32_t c = a; c > 0; --c) {
      const uint32_t lo = min(e[c - 1], e[c]), hi = max(e[c - 1], e[c]);
      e[c - 1] = lo;
      e[c] = hi;
    }
  if (nlow <= kLowBatch) {
    float4 r0[kLowBatch];
    float2 r1[kLowBatch];
#pragma unroll
    for (uint32_t p = 0; p < kLowBatch; ++p) {  // all loads in flight together
      const bool ok = p < nlow;
      const uint32_t i = e[p] >> 5, k = e[p] & 31u;
      r0[p] = ok ? __ldcs(&b.R0[(size_t)k * N + i]) : make_float4(0.f, 0.f, 0.f, 0.f);
      r1[p] = (ok && MODEL == 0) ? __ldcs(&b.R1[(size_t)k * N + i]) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (uint32_t p = 0; p < kLowBatch; ++p)
      if (p < nlow) add(r0[p], r1[p], -1.f);
  } else {  // more than kLowBatch lower contacts: selection in ascending order
    uint32_t prev = 0u;
    for (uint32_t r = 0; r < nlow; ++r) {
      uint32_t best = 0xFFFFFFFFu;
      for (uint32_t p = 0; p < nlow; ++p) {
        const uint32_t v = __ldcs(&b.llist[(size_t)p * N + j]);
        if ((r == 0 || v > prev) && v < best) best = v;
      }
      prev = best;
      const uint32_t i = best >> 5, k = best & 31u;
      add(__ldcs(&b.R0[(size_t)k * N + i]),
          MODEL == 0 ? __ldcs(&b.R1[(size_t)k * N + i]) : make_float2(0.f, 0.f), -1.f);
    }
  }
  // upper contacts: this particle's own results, candidate order
  for (uint32_t k0 = 0; k0 < nup; k0 += 4) {
    float4 r0[4];
    float2 r1[4];
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u) {
      const bool ok = k0 + u < nup;
      r0[u] = ok ? __ldcs(&b.R0[(size_t)(k0 + u) * N + j]) : make_float4(0.f, 0.f, 0.f, 0.f);
      r1[u] = (ok && MODEL == 0) ? __ldcs(&b.R1[(size_t)(k0 + u) * N + j]) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u)
      if (k0 + u < nup) add(r0[u], r1[u], 1.f);
  }
  auto lookup = [&](uint32_t pid) -> f3 {  // walls: after the pair contacts in the old list
    return old_history(b.hist_in, K, s, n_old, n_old, pid);
  };
  finish_particle<MODEL, DIAG, MAT>(b, g, ph, N, K, j - jlo, o, F, T, min(nup + nlow, K), overflow,
                               lookup);
}

#endif  // DEM_ABLATIONS

// Set the dynamic shared-memory limit of every k_force instantiation once,
// outside any stream capture (cudaFuncSetAttribute is not capturable).
#if DEM_FORCE_KC32
#define DEM_KC32_ATTR(MODEL, DIAG) cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, false, 32u>, A, sl);
#else
#define DEM_KC32_ATTR(MODEL, DIAG)
#endif
void sweep_prepare(uint32_t K) {
  const int sd = (int)(WarpSmemLayout::make(K, kForceDense).bytes * kSweepWarps);
  const int sl = (int)(WarpSmemLayout::make(K, kForceLight).bytes * kSweepWarps);
  const int fd = (int)(WarpSmemLayout::make(K, kForceDense, true).bytes * kSweepWarps);
  const int fl = (int)(WarpSmemLayout::make(K, kForceLight, true).bytes * kSweepWarps);
  const auto A = cudaFuncAttributeMaxDynamicSharedMemorySize;
#define DEM_SET_SMEM(MODEL, DIAG)                                     \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceDense, false>, A, sd); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceDense, true>, A, sd);  \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, false>, A, sl); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, true>, A, sl); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceDense, false, kForceKC>, A, sd); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, false, kForceKC>, A, sl); \
  DEM_KC32_ATTR(MODEL, DIAG)                                                        \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceDense, true, 0, true>, A, fd); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceDense, false, 0, true>, A, fd); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceDense, false, kForceKC, true>, A, fd); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, true, 0, true>, A, fl); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, false, 0, true>, A, fl); \
  cudaFuncSetAttribute(k_force<MODEL, DIAG, kForceLight, false, kForceKC, true>, A, fl);
  DEM_SET_SMEM(0, false)
  DEM_SET_SMEM(0, true)
  DEM_SET_SMEM(1, false)
  DEM_SET_SMEM(1, true)
#undef DEM_SET_SMEM
#if DEM_ABLATIONS
  const int sws = (int)(WsLayout::make(K).bytes * kWsPairs);
  cudaFuncSetAttribute(k_force_ws<0, false, false>, A, sws);
  cudaFuncSetAttribute(k_force_ws<0, false, true>, A, sws);
  cudaFuncSetAttribute(k_force_ws<0, true, false>, A, sws);
  cudaFuncSetAttribute(k_force_ws<0, true, true>, A, sws);
  cudaFuncSetAttribute(k_force_ws<1, false, false>, A, sws);
  cudaFuncSetAttribute(k_force_ws<1, false, true>, A, sws);
  cudaFuncSetAttribute(k_force_ws<1, true, false>, A, sws);
  cudaFuncSetAttribute(k_force_ws<1, true, true>, A, sws);
  cudaFuncSetAttribute(k_force_ws<0, false, false, kForceKC>, A, sws);
  cudaFuncSetAttribute(k_force_ws<0, true, false, kForceKC>, A, sws);
  cudaFuncSetAttribute(k_force_ws<1, false, false, kForceKC>, A, sws);
  cudaFuncSetAttribute(k_force_ws<1, true, false, kForceKC>, A, sws);
#endif
}

// --------------------------------------------------------- slab exchange --
// DESIGN.md §7. Slabs along z; each step ends with a deterministic pack of the
// output slots flagged by the integrator (migrants with their history, and the
// particles of the two boundary planes as the neighbours' ghosts) into this
// rank's exchange region, published with a system-scope release of the step
// tag; the next step starts by acquiring the neighbours' tags and appending
// their migrants and ghosts straight from peer memory (CUDA IPC over
// NVLink/NVSwitch, or the same device), in a fixed order (migrants from the
// left, from the right, ghosts from the left, from the right) so the stable
// sort that follows is deterministic.

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int global_cz(const DevGrid& g, float z) {
  return cell_coord(z, g.lo[2], g.inv_h, g.nz_global);
}

__global__ void k_keep(int64_t n, const float* pos, DevGrid g, uint32_t* keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cz = global_cz(g, pos[3 * i + 2]);
  keep[i] = (cz >= g.z0 && cz < g.z1) ? 1u : 0u;
}

// particles per global z-plane of the whole input set (identical on every
// rank given the same set: the exchange capacities derive from its maximum)
__global__ void k_plane_hist(int64_t n, const float* pos, DevGrid g, uint32_t* hist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  atomicAdd(&hist[global_cz(g, pos[3 * i + 2])], 1u);
}

__global__ void k_flags(int64_t n, const float4* pos, DevGrid g, uint32_t* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cz = global_cz(g, pos[i].z);
  flags[i] = (cz < g.z0 ? 1u : 0u) | (cz >= g.z1 ? 2u : 0u);  // (none: the set keeps owned ones)
}


__device__ __forceinline__ uint32_t owned_out(const StepBuffers& b, const DevGrid& g) {
  return __ldg(&b.off[g.own_c1]) - __ldg(&b.off[g.own_c0]);
}

// counts of the four categories per tile, for the state dem_set_particles
// publishes (in a step the integrator accumulates them: finish_particle)
__global__ void __launch_bounds__(256) k_xpack_count(StepBuffers b, DevGrid g, uint32_t* tc,
                                                     uint32_t ntiles, XState* xs) {
  __shared__ uint32_t s_c[4];
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t n_out = xs->n_out;
  if (threadIdx.x < 4) s_c[threadIdx.x] = 0;
  __syncthreads();
  uint32_t c[4] = {0, 0, 0, 0};
  for (int u = 0; u < 4; ++u) {
    const uint32_t o = blockIdx.x * kXTile + u * 256 + threadIdx.x;
    if (o < n_out) {
      const uint32_t f = b.flags[o];
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] += (f >> q) & 1u;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t v = c[q];
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane_id() == 0) atomicAdd(&s_c[q], v);
  }
  __syncthreads();
  if (threadIdx.x < 4) tc[threadIdx.x * ntiles + blockIdx.x] = s_c[threadIdx.x];
  if (threadIdx.x == 0) {
    const uint32_t sum = s_c[0] + s_c[1] + s_c[2] + s_c[3];
    tc[4 * ntiles + blockIdx.x] = sum;
    if (sum) atomicAdd(&tc[5 * ntiles], 1u);  // tiles with flagged outputs
  }
}

constexpr uint32_t kXPlaneMv = 1024;  // movers in or out of a boundary plane held in shared memory

// Step end: this rank's boundary plane (the first owned plane for the left
// neighbour, dir 0; the last for the right one) as the next step's sort will
// order it — the plane's stayers, minus the movers that left it, plus those
// that entered it, by k_merge's counts restricted to the plane's cells (the
// mover list is complete once the integrator is done) — with the new state
// and the plane's cell offsets relative to its first particle; its count in
// the header (the pack's last block releases the tag). Threads over the
// plane's previous slots, its entering movers and its cells.
struct PlaneSmem {
  uint4 in[kXPlaneMv];   // (key, slot, insertion point) of the entering movers
  uint2 out[kXPlaneMv];  // (previous slot, previous key) of the leaving ones
  uint32_t ni, no;
};

// (one block `pb` of the 2 x half plane blocks; returns without writing for
// a direction with no neighbour)
__device__ __forceinline__ void xpack_plane_block(const StepBuffers& b, const DevGrid& g,
                                                  uint8_t* mine, const XLayout& L, int nbr,
                                                  uint32_t pb, uint32_t half, PlaneSmem& sm) {
  uint4* s_in = sm.in;
  uint2* s_out = sm.out;
  uint32_t& s_ni = sm.ni;
  uint32_t& s_no = sm.no;
  const uint32_t tag = ld_volatile(&b.err->step_ctr) + 1u + g.xbase;  // the step that reads it
  const uint32_t par = tag & 1u;
  const uint32_t P = L.plane;
  const int dir = pb < half ? 0 : 1;
  if (!((nbr >> dir) & 1)) return;
  const uint32_t t = (pb - (dir ? half : 0)) * blockDim.x + threadIdx.x;
  const uint32_t cf = dir == 0 ? g.own_c0 : g.own_c1 - P;
  const uint32_t gl = b.gl_base;
  const uint32_t A = __ldg(&b.off[cf]) - gl, B = __ldg(&b.off[cf + P]) - gl;  // output slots
  if (threadIdx.x == 0) s_ni = s_no = 0u;
  __syncthreads();
  const uint32_t m = min(ld_volatile(b.mv.n_out), b.mv.cap);
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint4 v = __ldcg(&b.mv.list_out[i]);  // (a, c, c', x)
    if (v.w != 0xFFFFFFFFu && v.y - cf < P) {
      const uint32_t q = atomicAdd(&s_ni, 1u);
      if (q < kXPlaneMv) s_in[q] = make_uint4(v.y, v.x, v.w, 0u);
    }
    if (v.z - cf < P) {
      const uint32_t q = atomicAdd(&s_no, 1u);
      if (q < kXPlaneMv) s_out[q] = make_uint2(v.x, v.z);
    }
  }
  __syncthreads();
  const uint32_t ni = s_ni, no = s_no;
  uint8_t* blk = mine + (size_t)(dir * 2 + par) * L.bytes;
  const uint32_t n_new = (B - A) - no + ni;
  if (ni > kXPlaneMv || no > kXPlaneMv || n_new > L.ghost_cap) {
    if (t == 0) raise_error(b.err, 6u, cf, n_new);
    return;
  }
  if (t == 0) reinterpret_cast<XHeader*>(blk + L.header)->n_ghost = n_new;
  auto put = [&](uint32_t p, uint32_t s) {  // plane position p <- output slot s (new state)
    reinterpret_cast<float4*>(blk + L.gh_pos)[p] = __ldg(&b.pos_out[s]);
    reinterpret_cast<float4*>(blk + L.gh_vel)[p] = __ldg(&b.vel_out[s]);
    reinterpret_cast<float4*>(blk + L.gh_omg)[p] = __ldg(&b.omg_out[s]);
  };
  if (t < B - A) {  // a previous member: kept unless it left
    const uint32_t s = A + t;
    int d = 0;
    bool gone = false;
    for (uint32_t i = 0; i < ni; ++i) d += s_in[i].z <= s ? 1 : 0;
    for (uint32_t i = 0; i < no; ++i) {
      d -= s_out[i].x <= s ? 1 : 0;
      gone |= s_out[i].x == s;
    }
    if (!gone) put((uint32_t)((int)t + d), s);
  }
  if (t < ni) {  // an entering mover: its rank among them + the stayers before its point
    const uint4 mi = s_in[t];
    int r = 0;
    for (uint32_t i = 0; i < ni; ++i)
      r += (s_in[i].x < mi.x || (s_in[i].x == mi.x && s_in[i].y < mi.y)) ? 1 : 0;
    for (uint32_t i = 0; i < no; ++i) r -= s_out[i].x < mi.z ? 1 : 0;
    put((uint32_t)(r + (int)(mi.z - A)), mi.y);
  }
  if (t <= P) {  // the cell offsets, relative to the plane's first particle
    const uint32_t c = cf + t;
    int d = (int)(__ldg(&b.off[c]) - gl - A);
    for (uint32_t i = 0; i < ni; ++i) d += s_in[i].x < c ? 1 : 0;
    for (uint32_t i = 0; i < no; ++i) d -= s_out[i].y < c ? 1 : 0;
    reinterpret_cast<uint32_t*>(blk + L.gh_off)[t] = (uint32_t)d;
  }
}

__global__ void __launch_bounds__(256) k_xpack_planes(StepBuffers b, DevGrid g, uint8_t* mine,
                                                      XLayout L, int nbr) {
  __shared__ PlaneSmem sm;
  if (ld_volatile(&b.err->code) != 0u) return;
  if (threadIdx.x == 0) sm.ni = sm.no = 0u;
  __syncthreads();
  xpack_plane_block(b, g, mine, L, nbr, blockIdx.x, gridDim.x / 2, sm);
}

// deterministic placement: prefix over earlier tiles + in-tile rank (slot
// order); the last block to finish publishes the header counts and the tag
// (system-scope release). Each block clears its tile's counts of the other
// parity (the next step's integrator accumulates there).
// initial: the state dem_set_particles published (xs->n_out preset), else
// the step's owned outputs, recorded in xs->n_out for the next step's append.
__global__ void __launch_bounds__(256) k_xpack_write(StepBuffers b, DevGrid g, uint32_t K,
                                                     uint32_t N, uint8_t* mine, XLayout L,
                                                     const uint32_t* tc, uint32_t* tc_next,
                                                     uint32_t ntiles, XState* xs, int initial) {
  __shared__ uint32_t s_base[4];
  __shared__ uint32_t s_warp[4][8];
  __shared__ uint32_t s_cnt[4][32];  // [category][sub-tile * 8 + warp]
  __shared__ uint32_t s_last;
  // a failed step still publishes (a poisoned header, below), so that its
  // neighbours fail at once instead of waiting out the tag timeout: its
  // blocks skip the writes but take part in the publication count
  const bool failed = ld_volatile(&b.err->code) != 0u;
  const uint32_t writers = __ldcg(&tc[5 * ntiles]);  // tiles with flagged outputs
  const uint32_t tag = ld_volatile(&b.err->step_ctr) + 1u + g.xbase;  // the step that reads it
  const uint32_t par = tag & 1u;
  {
  const uint32_t n_out = initial ? xs->n_out : owned_out(b, g);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  // a tile without flagged outputs (all but the boundary planes' few) has
  // nothing to write: straight to the publication count
  const bool any = __ldcg(&tc[4 * ntiles + blockIdx.x]) != 0u;
  const bool work = any && !failed;
  // this tile's base per category: the counts of the earlier tiles, summed
  // block-wide (a serial sum by 4 threads cost ~100 us per step at 500 tiles)
  if (work) {
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    for (uint32_t t = threadIdx.x; t < blockIdx.x; t += blockDim.x)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += tc[q * ntiles + t];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      for (int d = 16; d > 0; d >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], d);
      if (lane == 0) s_warp[q][warp] = acc[q];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      uint32_t s = 0;
      for (int w = 0; w < 8; ++w) s += s_warp[threadIdx.x][w];
      s_base[threadIdx.x] = s;
    }
    __syncthreads();
  }
  if (work) {
    // the tile's four sub-tiles at once (their loads in flight together): a
    // flagged output's rank in its category = this tile's base + the flagged
    // outputs before it in slot order (sub-tile, warp, lane)
    uint32_t f[4], rk[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t o = blockIdx.x * kXTile + u * 256 + threadIdx.x;
      f[u] = o < n_out ? __ldcg(&b.flags[o]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t m = __ballot_sync(0xffffffffu, (f[u] >> q) & 1u);
        rk[u][q] = __popc(m & lanemask_lt());
        if (lane == 0) s_cnt[q][u * 8 + warp] = __popc(m);
      }
    __syncthreads();
    if (threadIdx.x < 4) {  // exclusive prefix over (sub-tile, warp), per category
      uint32_t acc = s_base[threadIdx.x];
      for (int w = 0; w < 32; ++w) {
        const uint32_t c = s_cnt[threadIdx.x][w];
        s_cnt[threadIdx.x][w] = acc;
        acc += c;
      }
    }
    __syncthreads();
    float4 P[4], V[4], W[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t o = blockIdx.x * kXTile + u * 256 + threadIdx.x;
      if (f[u]) {
        P[u] = __ldcg(&b.pos_out[o]);
        V[u] = __ldcg(&b.vel_out[o]);
        W[u] = __ldcg(&b.omg_out[o]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!f[u]) continue;
      const uint32_t o = blockIdx.x * kXTile + u * 256 + threadIdx.x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!((f[u] >> q) & 1u)) continue;
        const int dir = q & 1;  // 0: to the left neighbour, 1: to the right
        uint8_t* blk = mine + (size_t)(dir * 2 + par) * L.bytes;
        const uint32_t e = s_cnt[q][u * 8 + warp] + rk[u][q];
        if (q < 2) {  // migrant: state + history
          if (e >= L.mig_cap) {
            raise_error(b.err, 6u, o, __float_as_uint(W[u].w));
            continue;
          }
          reinterpret_cast<float4*>(blk + L.mig_pos)[e] = P[u];
          reinterpret_cast<float4*>(blk + L.mig_vel)[e] = V[u];
          reinterpret_cast<float4*>(blk + L.mig_omg)[e] = W[u];
          const uint32_t nc = b.cnt_out[o];
          reinterpret_cast<uint32_t*>(blk + L.mig_cnt)[e] = nc;
          float4* h = reinterpret_cast<float4*>(blk + L.mig_hist) + (size_t)e * K;
          for (uint32_t k = 0; k < nc; ++k) h[k] = b.hist_out[hix(o, k, K)];
        } else {  // ghost: state only
          if (e >= L.ghost_cap) {
            raise_error(b.err, 6u, o, __float_as_uint(W[u].w));
            continue;
          }
          reinterpret_cast<float4*>(blk + L.gh_pos)[e] = P[u];
          reinterpret_cast<float4*>(blk + L.gh_vel)[e] = V[u];
          reinterpret_cast<float4*>(blk + L.gh_omg)[e] = W[u];
        }
      }
    }
    __syncthreads();
  }
  // the next step's counts start from zero (this tile's, and the tile count)
  if (threadIdx.x < 5) tc_next[threadIdx.x * ntiles + blockIdx.x] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) tc_next[5 * ntiles] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0 && !initial) xs->n_out = n_out;
  // publication by the last of the `writers` blocks that wrote (block 0 when
  // none did). A block's records are ordered before its count (block
  // barrier, then a gpu-scope fence); the publisher's system-scope release
  // fence is cumulative over them
  if (threadIdx.x == 0) {
    s_last = 0u;
    if (any) {
      __threadfence();
      s_last = atomicAdd(&xs->done, 1u) == writers - 1u ? 1u : 0u;
    } else if (writers == 0u && blockIdx.x == 0) {
      s_last = 1u;
    }
  }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the category totals over all tiles, block-wide
  uint32_t tot[4] = {0, 0, 0, 0};
  for (uint32_t t = threadIdx.x; t < ntiles; t += blockDim.x)
#pragma unroll
    for (int q = 0; q < 4; ++q) tot[q] += __ldcg(&tc[q * ntiles + t]);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    for (int d = 16; d > 0; d >>= 1) tot[q] += __shfl_xor_sync(0xffffffffu, tot[q], d);
    if ((threadIdx.x & 31u) == 0u) s_warp[q][threadIdx.x >> 5] = tot[q];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  xs->done = 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    tot[q] = 0;
    for (int w = 0; w < 8; ++w) tot[q] += s_warp[q][w];
  }
  // poisoned when this rank's step failed (its error word, any block's
  // overflow included) or more migrants left than a block holds
  const bool poison = ld_volatile(&b.err->code) != 0u || tot[0] > L.mig_cap || tot[1] > L.mig_cap;
  XHeader* h[2];
  for (int dir = 0; dir < 2; ++dir) {
    h[dir] = reinterpret_cast<XHeader*>(mine + (size_t)(dir * 2 + par) * L.bytes + L.header);
    h[dir]->n_mig = poison ? kXPoison : tot[dir];  // (n_ghost: k_xpack_planes / k_xplanes_initial)
  }
  // one system-scope release fence for both tags (a fence.sc.sys + st.release.sys
  // per tag, as before, was four system membars: ~15 us of a 20 us pack)
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int dir = 0; dir < 2; ++dir)
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(&h[dir]->tag), "r"(tag) : "memory");
}

// Thread-level acquire of a neighbour's tag, bounded (~30 s): a dead
// neighbour becomes DEM_EPEER instead of a hang. false on time-out.
__device__ __forceinline__ bool wait_tag(const uint32_t* t, uint32_t want, uint32_t* seen) {
  unsigned long long spins = 0;
  uint32_t v;
  while ((v = ld_acquire_sys(t)) != want) {
    if (++spins > (1ull << 27)) {
      *seen = v;
      return false;
    }
    __nanosleep(200);
  }
  return true;
}

// Step start: every block acquires the neighbours' tags (thread 0 the left
// neighbour's block "to the right", thread 1 the right one's "to the left"),
// then appends their migrants (state + tangential history) at slots n_out..,
// left first, in the senders' slot order, hashed — a merge step lists each as
// an insertion for k_merge (new key, previous key 0xFFFFFFFF, insertion point
// the end of its cell in the last order), a counting step counts it into its
// cell — and after them the state of their boundary planes (left, then
// right), which k_xghost_place sorts in. Block 0 records the counts and the
// input slots the sort takes (owned outputs + migrants).
__global__ void __launch_bounds__(256) k_xrecv(StepBuffers b, DevGrid g, uint32_t K, uint32_t N,
                                               const uint8_t* left, const uint8_t* right,
                                               XLayout L, XState* xs, uint32_t* nslots, int merge) {
  __shared__ uint32_t s_cnt[4], s_seen[2];
  __shared__ uint32_t s_ok, s_bad;
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t tag = ld_volatile(&b.err->step_ctr) + 1u + g.xbase;
  const uint32_t par = tag & 1u;
  if (threadIdx.x == 0) {
    s_ok = 1u;
    s_bad = 0u;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    const uint8_t* peer = threadIdx.x == 0 ? left : right;
    const int dir = threadIdx.x == 0 ? 1 : 0;
    uint32_t nm = 0, ng = 0;
    if (peer) {
      const XHeader* h =
          reinterpret_cast<const XHeader*>(peer + (size_t)(dir * 2 + par) * L.bytes + L.header);
      if (!wait_tag(&h->tag, tag, &s_seen[threadIdx.x])) s_ok = 0u;
      nm = ld_volatile(&h->n_mig);
      ng = ld_volatile(&h->n_ghost);
      // the neighbour's step failed (kXPoison), or counts past the blocks
      if (nm > L.mig_cap || ng > L.ghost_cap) {
        s_bad = 1u;
        nm = ng = 0u;
      }
    }
    s_cnt[threadIdx.x] = nm;
    s_cnt[2 + threadIdx.x] = ng;
  }
  __syncthreads();
  const uint32_t c0 = s_cnt[0], c1 = s_cnt[1], c2 = s_cnt[2], c3 = s_cnt[3];
  const uint32_t tot = c0 + c1 + c2 + c3;
  const uint32_t base = xs->n_out;
  if (s_ok && s_bad) {  // slot 0xFFFFFE00: a neighbour published a failed step
    if (threadIdx.x == 0) raise_error(b.err, 11u, 0xFFFFFE00u, 0u);
    return;
  }
  if (!s_ok) {  // slot: 0xFFFFFF00 | expected tag's low byte; id: tags seen (left, right)
    if (threadIdx.x == 0)
      raise_error(b.err, 11u, 0xFFFFFF00u | (tag & 0xFFu),
                  ((s_seen[0] & 0xFFFFu) << 16) | (s_seen[1] & 0xFFFFu));
    return;
  }
  if ((uint64_t)base + tot > N) {
    if (threadIdx.x == 0) raise_error(b.err, 6u, base, 0u);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) xs->appended[q] = s_cnt[q];
    xs->pad[0] = tag;  // this step's tag (k_merge's ghost blocks take its parity)
    *nslots = base + c0 + c1;
  }
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tot) return;
  uint32_t q, e;
  if (i < c0) { q = 0; e = i; }
  else if (i < c0 + c1) { q = 1; e = i - c0; }
  else if (i < c0 + c1 + c2) { q = 2; e = i - c0 - c1; }
  else { q = 3; e = i - c0 - c1 - c2; }
  const bool from_left = (q & 1u) == 0u;
  const uint8_t* blk = (from_left ? left : right) + (size_t)((from_left ? 1 : 0) * 2 + par) * L.bytes;
  const uint32_t slot = base + i;
  float4 P, V, W;
  if (q < 2) {
    P = __ldcv(reinterpret_cast<const float4*>(blk + L.mig_pos) + e);
    V = __ldcv(reinterpret_cast<const float4*>(blk + L.mig_vel) + e);
    W = __ldcv(reinterpret_cast<const float4*>(blk + L.mig_omg) + e);
    const uint32_t nc = min(__ldcv(reinterpret_cast<const uint32_t*>(blk + L.mig_cnt) + e), K);
    const float4* h = reinterpret_cast<const float4*>(blk + L.mig_hist) + (size_t)e * K;
    float4* hist = const_cast<float4*>(b.hist_in);
    for (uint32_t k = 0; k < nc; ++k) hist[hix(slot, k, K)] = __ldcv(h + k);
    const_cast<uint32_t*>(b.cnt_in)[slot] = nc;
  } else {
    P = __ldcv(reinterpret_cast<const float4*>(blk + L.gh_pos) + e);
    V = __ldcv(reinterpret_cast<const float4*>(blk + L.gh_vel) + e);
    W = __ldcv(reinterpret_cast<const float4*>(blk + L.gh_omg) + e);
    const_cast<uint32_t*>(b.cnt_in)[slot] = 0u;
  }
  const_cast<float4*>(b.pos_in)[slot] = P;
  const_cast<float4*>(b.vel_in)[slot] = V;
  const_cast<float4*>(b.omg_in)[slot] = W;
  if (q >= 2) return;  // (ghosts: placed by k_xghost_place in the senders' sorted order)
  const uint32_t k2 = cell_key(g, P.x, P.y, P.z);
  // a migrant must land in this rank's owned planes (one plane per step)
  const int cz = global_cz(g, P.z);
  if (cz < g.z0 || cz >= g.z1) {
    raise_error(b.err, 11u, slot, __float_as_uint(W.w));
    return;
  }
  const_cast<uint32_t*>(b.key_in)[slot] = k2;
  if (merge) {
    // where one sorted order of all the particles puts it: an arrival from
    // the left came from earlier slots (first in its cell, before the cell's
    // movers: previous key 0xFFFFFFFE ranks it first), one from the right
    // from later slots (last in its cell)
    const uint32_t idx = atomicAdd(const_cast<uint32_t*>(b.mv.n_in), 1u);  // (order-free counts)
    if (idx < b.mv.cap)
      const_cast<uint4*>(b.mv.list_in)[idx] =
          from_left ? make_uint4(slot, k2, 0xFFFFFFFEu, __ldg(&b.off[k2]) - b.gl_base)
                    : make_uint4(slot, k2, 0xFFFFFFFFu, __ldg(&b.off[k2 + 1]) - b.gl_base);
  } else {
    b.prank[slot] = count_into_cell(b.count, k2);
  }
}

// (after a counting sort: the owned particles are placed, off[own_c1] is set)
__global__ void __launch_bounds__(256) k_xghost_place(StepBuffers b, DevGrid g, uint32_t N,
                                                      const uint8_t* left, const uint8_t* right,
                                                      XLayout L, XState* xs) {
  __shared__ GhostSmem sm;
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t tag = ld_volatile(&b.err->step_ctr) + g.xbase;  // (the sort counted this step)
  ghost_place_block(b, g, N, left, right, L, xs, tag & 1u, blockIdx.x, gridDim.x / 2, false, 0u,
                    sm);
}

// The set state's boundary planes (dem_set_particles sorts it by counting
// before publishing): each plane is a sorted run of pos_sorted, its state in
// the set arrays (b.*_out here) through the old slot; the cell offsets
// relative to the run's start.
__global__ void __launch_bounds__(256) k_xplanes_initial(StepBuffers b, DevGrid g, uint8_t* mine,
                                                         XLayout L, int nbr) {
  if (ld_volatile(&b.err->code) != 0u) return;
  const uint32_t tag = ld_volatile(&b.err->step_ctr) + 1u + g.xbase;
  const uint32_t par = tag & 1u;
  const uint32_t P = L.plane;
  const uint32_t half = gridDim.x / 2;
  const int dir = blockIdx.x < half ? 0 : 1;
  if (!((nbr >> dir) & 1)) return;
  const uint32_t t = (blockIdx.x - (dir ? half : 0)) * blockDim.x + threadIdx.x;
  const uint32_t cf = dir == 0 ? g.own_c0 : g.own_c1 - P;
  const uint32_t lo = __ldg(&b.off[cf]), hi = __ldg(&b.off[cf + P]);
  uint8_t* blk = mine + (size_t)(dir * 2 + par) * L.bytes;
  if (hi - lo > L.ghost_cap) {
    if (t == 0) raise_error(b.err, 6u, cf, hi - lo);
    return;
  }
  if (t == 0) reinterpret_cast<XHeader*>(blk + L.header)->n_ghost = hi - lo;
  const bool sw = b.sw_r > 0.f;
  if (t < hi - lo) {
    float4 Pp = __ldg(&b.pos_sorted[lo + t]);
    const uint32_t s = sw ? __float_as_uint(Pp.w) : __ldg(&b.perm[lo + t]);
    reinterpret_cast<float4*>(blk + L.gh_pos)[t] = __ldg(&b.pos_out[s]);
    reinterpret_cast<float4*>(blk + L.gh_vel)[t] = __ldg(&b.vel_out[s]);
    reinterpret_cast<float4*>(blk + L.gh_omg)[t] = __ldg(&b.omg_out[s]);
  }
  if (t <= P) reinterpret_cast<uint32_t*>(blk + L.gh_off)[t] = __ldg(&b.off[cf + t]) - lo;
}

// --------------------------------------------------- introspection ---------

__global__ void k_unpack(int64_t n, bool by_id, const float4* pos, const float4* vel,
                         const float4* omg, const float4* F, const float4* T, float* o_pos,
                         float* o_vel, float* o_omg, float* o_r, float* o_m, uint32_t* o_id,
                         float* o_F, float* o_T, uint32_t idmask, uint32_t* o_mat) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 P = pos[i], V = vel[i], W = omg[i];
  const uint32_t word = __float_as_uint(W.w);
  const uint32_t id = word & idmask;
  const int64_t d = by_id ? (int64_t)id : i;
  if (o_pos) { o_pos[3 * d] = P.x; o_pos[3 * d + 1] = P.y; o_pos[3 * d + 2] = P.z; }
  if (o_vel) { o_vel[3 * d] = V.x; o_vel[3 * d + 1] = V.y; o_vel[3 * d + 2] = V.z; }
  if (o_omg) { o_omg[3 * d] = W.x; o_omg[3 * d + 1] = W.y; o_omg[3 * d + 2] = W.z; }
  if (o_r) o_r[d] = P.w;
  if (o_m) o_m[d] = V.w;
  if (o_id) o_id[d] = id;
  if (o_mat) o_mat[d] = idmask == 0xFFFFFFFFu ? 0u : (word >> kMatShift);
  if (o_F && F) { float4 f = F[i]; o_F[3 * d] = f.x; o_F[3 * d + 1] = f.y; o_F[3 * d + 2] = f.z; }
  if (o_T && T) { float4 t = T[i]; o_T[3 * d] = t.x; o_T[3 * d + 1] = t.y; o_T[3 * d + 2] = t.z; }
}

__global__ void k_emit_contacts(int64_t n, int64_t stride, uint32_t K, const float4* hist,
                                const uint32_t* cnt, const uint32_t* base, const float4* omg,
                                uint32_t* id_i, uint32_t* id_j, float* dt3, uint32_t idmask) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cnt[i], o = base[i];
  const uint32_t me = __float_as_uint(omg[i].w) & idmask;
  for (uint32_t k = 0; k < c && k < K; ++k) {
    const float4 h = hist[hix(i, k, K)];
    if (id_i) id_i[o + k] = me;
    if (id_j) id_j[o + k] = __float_as_uint(h.w);
    if (dt3) { dt3[3 * (o + k)] = h.x; dt3[3 * (o + k) + 1] = h.y; dt3[3 * (o + k) + 2] = h.z; }
  }
}

__global__ void k_slot_of_id(int64_t n, uint32_t idmask, const float4* omg, uint32_t* slot_of_id) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  slot_of_id[__float_as_uint(omg[i].w) & idmask] = (uint32_t)i;
}

// flags[0] |= 1: id out of range, |= 2: capacity overflow. slot_of_id has
// id_bound entries; 0xFFFFFFFF marks an id this handle does not hold (a slab
// rank skips the contacts of other ranks' particles).
__global__ void k_insert_contacts(int64_t m, int64_t id_bound, int64_t stride, uint32_t K,
                                  const uint32_t* id_i,
                                  const uint32_t* id_j, const float* dt3,
                                  const uint32_t* slot_of_id, float4* hist, uint32_t* cnt,
                                  uint32_t* flags, int skip_unknown) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const uint32_t a = id_i[e];
  if (a >= (uint64_t)id_bound) {
    if (!skip_unknown) atomicOr(flags, 1u);
    return;
  }
  const uint32_t s = slot_of_id[a];
  if (s == 0xFFFFFFFFu) return;
  const uint32_t k = atomicAdd(&cnt[s], 1u);
  if (k >= K) { atomicOr(flags, 2u); return; }
  hist[hix(s, k, K)] = make_float4(dt3[3 * e], dt3[3 * e + 1], dt3[3 * e + 2],
                                        __uint_as_float(id_j[e]));
}

// max |v| over n particles (bits of a non-negative float order like the value)
__global__ void k_max_speed(int64_t n, const float4* vel, uint32_t* out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = vel[i];
    m = fmaxf(m, sqrtf(v.x * v.x + v.y * v.y + v.z * v.z));
  }
  for (int d = 16; d > 0; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, d));
  if (lane_id() == 0) atomicMax(out, __float_as_uint(m));
}

__global__ void k_cnt_stats(int64_t n, const uint32_t* cnt, unsigned long long* sum_max) {
  unsigned long long s = 0;
  uint32_t mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    s += cnt[i];
    mx = max(mx, cnt[i]);
  }
  for (int d = 16; d > 0; d >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, d);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  }
  if (lane_id() == 0) {
    atomicAdd(&sum_max[0], s);
    atomicMax(&sum_max[1], (unsigned long long)mx);
  }
}

// §6 analysis (dem_analyze): per owned sorted slot of the last step, the
// candidate count of its 9 rows (Eq. 12) and its contact count, reduced per
// warp of 32 consecutive slots (the paper's mapping), plus the population of
// its cell. acc: [0] n, [1] Σcand, [2] max cand, [3] Σcont, [4] max cont,
// [5] Σ 32·warp-max cand, [6] Σ 32·warp-max cont, [7] max per cell,
// [8] occupied cells, [9..41] contact histogram.
__global__ void __launch_bounds__(256) k_analyze(StepBuffers b, DevGrid g, uint32_t N,
                                                 unsigned long long* acc) {
  __shared__ unsigned long long s_hist[33];
  if (threadIdx.x < 33) s_hist[threadIdx.x] = 0ull;
  __syncthreads();
  uint32_t jlo, jhi;
  owned_range(b, g, N, jlo, jhi);
  const uint32_t j = jlo + blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = j < jhi;
  uint32_t cand = 0, cont = 0, pop = 0, first = 0;
  if (valid) {
    float4 P = __ldg(&b.pos_sorted[j]);
    if (b.sw_r > 0.f) P.w = b.sw_r;  // (.w holds the old slot then)
    const int cx = cell_coord(P.x, g.lo[0], g.inv_h, g.nx);
    const int cy = cell_coord(P.y, g.lo[1], g.inv_h, g.ny);
    const int cz = cell_coord(P.z, g.lo[2], g.inv_h, g.nz_global) - g.zlo;
    const uint32_t xa = cx > 0 ? (uint32_t)cx - 1u : 0u;
    const uint32_t xb = cx < g.nx - 1 ? (uint32_t)cx + 1u : (uint32_t)g.nx - 1u;
    const uint32_t nxy = (uint32_t)g.nx * (uint32_t)g.ny;
    for (int dz = -1; dz <= 1; ++dz) {
      const int z = cz + dz;
      if (z < 0 || z >= g.nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g.ny) continue;
        const uint32_t row = (uint32_t)z * nxy + (uint32_t)y * (uint32_t)g.nx;
        const uint32_t t0 = __ldg(&b.off[row + xa]), t1 = __ldg(&b.off[row + xb + 1]);
        cand += t1 - t0;
        // contacts with the exact predicate (R14), independent of which force
        // path ran (the ablations keep no full contact counts)
        for (uint32_t t = t0; t < t1; ++t)
          if (t != j) {
            float4 Q = __ldg(&b.pos_sorted[t]);
            if (b.sw_r > 0.f) Q.w = b.sw_r;
            if (in_contact(P, Q)) ++cont;
          }
      }
    }
    cand -= 1u;  // itself
    const uint32_t c = (uint32_t)cz * nxy + (uint32_t)cy * (uint32_t)g.nx + (uint32_t)cx;
    const uint32_t o0 = __ldg(&b.off[c]);
    pop = __ldg(&b.off[c + 1]) - o0;
    first = (j == o0) ? 1u : 0u;
    atomicAdd(&s_hist[min(cont, 32u)], 1ull);
  }
  const uint32_t wmax_c = __reduce_max_sync(0xffffffffu, cand);
  const uint32_t wmax_k = __reduce_max_sync(0xffffffffu, cont);
  const uint32_t wpop = __reduce_max_sync(0xffffffffu, pop);
  const uint32_t wn = __reduce_add_sync(0xffffffffu, valid ? 1u : 0u);
  const uint32_t wcand = __reduce_add_sync(0xffffffffu, cand);
  const uint32_t wcont = __reduce_add_sync(0xffffffffu, cont);
  const uint32_t wfirst = __reduce_add_sync(0xffffffffu, first);
  if (lane_id() == 0 && wn > 0) {
    atomicAdd(&acc[0], (unsigned long long)wn);
    atomicAdd(&acc[1], (unsigned long long)wcand);
    atomicMax(&acc[2], (unsigned long long)wmax_c);
    atomicAdd(&acc[3], (unsigned long long)wcont);
    atomicMax(&acc[4], (unsigned long long)wmax_k);
    atomicAdd(&acc[5], 32ull * wmax_c);
    atomicAdd(&acc[6], 32ull * wmax_k);
    atomicMax(&acc[7], (unsigned long long)wpop);
    atomicAdd(&acc[8], (unsigned long long)wfirst);
  }
  __syncthreads();
  if (threadIdx.x < 33 && s_hist[threadIdx.x]) atomicAdd(&acc[9 + threadIdx.x], s_hist[threadIdx.x]);
}

// ------------------------------------------------------------ launchers ----

bool ablations_built() { return DEM_ABLATIONS != 0; }

static inline unsigned blocks_for(int64_t n, int threads) {
  return (unsigned)((n + threads - 1) / threads);
}

int launch_probe(cudaStream_t st, int64_t n, PackIn in, DevGrid g, Probe* out) {
  if (n <= 0) return K_OTHER;
  k_probe<<<blocks_for(n, 256), 256, 0, st>>>(n, in, g, out);
  return K_OTHER;
}

int launch_pack(cudaStream_t st, int64_t n, PackIn in, DevGrid g, float4* pos, float4* vel,
                float4* omg, uint32_t* key, uint32_t* count, uint32_t* prank, const uint32_t* dst,
                const uint32_t* keep) {
  if (n <= 0) return K_HASH;
  k_pack<<<blocks_for(n, 256), 256, 0, st>>>(n, in, g, pos, vel, omg, key, count, prank, dst,
                                              keep);
  return K_HASH;
}

int launch_count(cudaStream_t st, int64_t n, const uint32_t* key, uint32_t* count,
                 uint32_t* prank) {
  if (n <= 0) return K_HASH;
  k_count<<<blocks_for(n, 256), 256, 0, st>>>(n, key, count, prank);
  return K_HASH;
}

int launch_idcheck(cudaStream_t st, int64_t n, uint32_t idmask, const float4* omg, uint32_t* seen,
                   uint32_t* dup_flag) {
  if (n <= 0) return K_OTHER;
  k_idcheck<<<blocks_for(n, 256), 256, 0, st>>>(n, idmask, omg, seen, dup_flag);
  return K_OTHER;
}

// Launch with programmatic stream serialization (the kernel calls pdl_enter()).
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = DEM_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int launch_scan(cudaStream_t st, const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* zero,
                unsigned long long* status, uint32_t* ctr, DevErr* err, int count_step,
                uint32_t base0) {
  // `status` holds at least ceil(n / kScanTile) words: used as the tile sums
  (void)ctr;
  const unsigned tiles = (unsigned)((n + kScanTile - 1) / kScanTile);
  uint32_t* tsum = reinterpret_cast<uint32_t*>(status);
  launch_pdl(k_tile_sum, tiles > 0 ? tiles : 1, kScanThreads, 0, st, in, n, tsum, err, count_step);
  launch_pdl(k_scan_apply, tiles > 0 ? tiles : 1, kScanThreads, 0, st, in, out, n, zero,
             (const uint32_t*)tsum, err, base0);
  return K_SCAN;
}

int launch_scatter(cudaStream_t st, int64_t n, const StepBuffers& b) {
  const int64_t per = 256 * kItems;
  int64_t blocks = (n + per - 1) / per;
  if (blocks < 1) blocks = 1;
  launch_pdl(k_scatter, (unsigned)blocks, 256, 0, st, n, b.nslots, b.key_in, b.prank, b.off, b.tmp,
             b.err);
  return K_SCATTER;
}

int launch_rank(cudaStream_t st, int64_t n, const StepBuffers& b) {
  if (n <= 0) return K_RANK;
  const int64_t per = 256 * kItems;
  launch_pdl(k_rank, (unsigned)((n + per - 1) / per), 256, 0, st, n, b.key_in, b.off, b.tmp, b.perm,
             b.pos_in, b.pos_sorted, b.nslots, b.err, b.sw_r > 0.f, b.gl_base);
  return K_RANK;
}

int launch_merge(cudaStream_t st, int64_t n, uint32_t ncells, const StepBuffers& b,
                 const DevGrid& g, const uint32_t* n_dev, const uint8_t* left,
                 const uint8_t* right, const XLayout* L, XState* xs) {
  const int64_t span = n > (int64_t)ncells + 1 ? n : (int64_t)ncells + 1;
  unsigned grid = (unsigned)((span + kMergeSpan - 1) / kMergeSpan);
  // (slab: off[own_c1], the owned particles' end, is written by the ghost
  // blocks, which count it from the list: the merge blocks leave it alone)
  const uint32_t c_lo = g.slab ? g.own_c0 : 0u, c_hi = g.slab ? g.own_c1 - (L ? 1u : 0u) : ncells;
  GhostArgs ga{};
  if (L) {  // slab ranks: the ghost planes' blocks after the merge's
    ga.b = b;
    ga.g = g;
    ga.left = left;
    ga.right = right;
    ga.L = *L;
    ga.xs = xs;
    ga.N = (uint32_t)n;
    ga.nghost = 2 * ((L->plane + 1 + 255) / 256);
    grid += ga.nghost;
  }
  if (L)
    launch_pdl(k_merge<true>, grid, 256, 0, st, (uint32_t)n, ncells, b.mv, b.pos_in, b.perm,
               b.pos_sorted, b.off, b.err, b.sw_r > 0.f, n_dev, b.gl_base, c_lo, c_hi, ga);
  else
    launch_pdl(k_merge<false>, grid, 256, 0, st, (uint32_t)n, ncells, b.mv, b.pos_in, b.perm,
               b.pos_sorted, b.off, b.err, b.sw_r > 0.f, n_dev, b.gl_base, c_lo, c_hi, ga);
  return K_RANK;
}

// SCCM from the sorted positions' .w (one-radius path, where k_mv_apply
// keeps the old slot there instead of writing perm): dem_get_grid only
__global__ void k_perm_from_w(int64_t n, const float4* __restrict__ pos_sorted,
                              uint32_t* __restrict__ perm) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) perm[j] = __float_as_uint(pos_sorted[j].w);
}

int launch_perm_from_w(cudaStream_t st, int64_t n, const float4* pos_sorted, uint32_t* perm) {
  if (n > 0) k_perm_from_w<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, pos_sorted, perm);
  return 0;
}


template <int MODEL, bool DIAG>
static void sweep_dispatch(cudaStream_t st, int64_t n, uint32_t K, const StepBuffers& b,
                           const DevGrid& g, const DevPhys& ph, int variant) {
  const uint32_t N = (uint32_t)n;
  if (variant == 1 || variant == 4) {
#if DEM_ABLATIONS
  if (variant == 1) {  // the paper's mapping, one fused kernel
    if (ph.nmat > 1 || ph.nplates > 0)
      launch_pdl(k_sweep_tpp<MODEL, DIAG, true>, blocks_for(n, 128), 128, 0, st, b, g, ph, N, K);
    else
      launch_pdl(k_sweep_tpp<MODEL, DIAG, false>, blocks_for(n, 128), 128, 0, st, b, g, ph, N, K);
  } else if (variant == 4) {  // full contact lists, one lane per particle
    const unsigned grid = blocks_for(n, kLanesThreads);
    const bool mat = ph.nmat > 1 || ph.nplates > 0;
    if (mat) launch_pdl(k_force_lane<MODEL, DIAG, true>, grid, kLanesThreads, 0, st, b, g, ph, N, K);
    else if (K == kForceKC) launch_pdl(k_force_lane<MODEL, DIAG, false, kForceKC>, grid, kLanesThreads, 0, st, b, g, ph, N, K);
    else launch_pdl(k_force_lane<MODEL, DIAG, false>, grid, kLanesThreads, 0, st, b, g, ph, N, K);
  }
#endif
#if DEM_ABLATIONS
  } else if (variant == 5) {  // warp-specialised (DEM_F_FORCE_WS, ablation)
    const bool mat = ph.nmat > 1 || ph.nplates > 0;
    const uint32_t smem = WsLayout::make(K).bytes * kWsPairs;
    auto kern = mat ? k_force_ws<MODEL, DIAG, true>
                    : K == kForceKC ? k_force_ws<MODEL, DIAG, false, kForceKC> : k_force_ws<MODEL, DIAG, false>;
    int resident = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, 32 * 2 * kWsPairs, smem);
    if (resident < 1) resident = 1;
    const int64_t groups = (n + 31) / 32;
    int64_t grid = (int64_t)resident * sms;
    if (grid * kWsPairs > groups) grid = (groups + kWsPairs - 1) / kWsPairs;
    launch_pdl(kern, (unsigned)grid, 32 * 2 * kWsPairs, smem, st, b, g, ph, N, K);
#endif
  } else if (variant >= 6) {  // fused detection + warp-flattened rounds (6: dense, 7: light)
    const int cfg = variant == 7 ? kForceLight : kForceDense;
    const uint32_t smem = WarpSmemLayout::make(K, cfg, true).bytes * kSweepWarps;
    const unsigned grid = blocks_for(n, 32 * kSweepWarps), block = 32 * kSweepWarps;
    const bool mat = ph.nmat > 1 || ph.nplates > 0;
    const bool k16 = K == kForceKC;
#define DEM_FUSED(CFG)                                                                          \
  (mat ? launch_pdl(k_force<MODEL, DIAG, CFG, true, 0, true>, grid, block, smem, st, b, g, ph, N, K) \
   : k16 ? launch_pdl(k_force<MODEL, DIAG, CFG, false, kForceKC, true>, grid, block, smem, st, b, g, ph, N, K) \
         : launch_pdl(k_force<MODEL, DIAG, CFG, false, 0, true>, grid, block, smem, st, b, g, ph, N, K))
    if (cfg == kForceLight) DEM_FUSED(kForceLight);
    else DEM_FUSED(kForceDense);
#undef DEM_FUSED
  } else {  // full contact lists, warp-flattened contact rounds (2: dense, 3: light)
    const int cfg = variant == 3 ? kForceLight : kForceDense;
    const uint32_t smem = WarpSmemLayout::make(K, cfg).bytes * kSweepWarps;
    const unsigned grid = blocks_for(n, 32 * kSweepWarps), block = 32 * kSweepWarps;
    const bool mat = ph.nmat > 1 || ph.nplates > 0;  // materials/plates: their own instantiation
    const bool k16 = K == kForceKC;  // the default capacity: compile-time K
    if (cfg == kForceLight) {
      if (mat) launch_pdl(k_force<MODEL, DIAG, kForceLight, true>, grid, block, smem, st, b, g, ph, N, K);
      else if (k16) launch_pdl(k_force<MODEL, DIAG, kForceLight, false, kForceKC>, grid, block, smem, st, b, g, ph, N, K);
#if DEM_FORCE_KC32
      else if (K == 32u) launch_pdl(k_force<MODEL, DIAG, kForceLight, false, 32u>, grid, block, smem, st, b, g, ph, N, K);
#endif
      else launch_pdl(k_force<MODEL, DIAG, kForceLight, false>, grid, block, smem, st, b, g, ph, N, K);
    } else {
      if (mat) launch_pdl(k_force<MODEL, DIAG, kForceDense, true>, grid, block, smem, st, b, g, ph, N, K);
      else if (k16) launch_pdl(k_force<MODEL, DIAG, kForceDense, false, kForceKC>, grid, block, smem, st, b, g, ph, N, K);
      else launch_pdl(k_force<MODEL, DIAG, kForceDense, false>, grid, block, smem, st, b, g, ph, N, K);
    }
  }
}

int launch_detect_half(cudaStream_t st, int64_t n, uint32_t K, const StepBuffers& b,
                       const DevGrid& g) {
#if DEM_ABLATIONS
  if (n <= 0) return K_DETECT;
  cudaMemsetAsync(b.lcount, 0, sizeof(uint32_t) * n, st);
  k_detect_half<<<blocks_for(n, 256), 256, 0, st>>>(b, g, (uint32_t)n, K);
#endif
  return K_DETECT;
}

int launch_pair(cudaStream_t st, int64_t n, uint32_t K, int model, const StepBuffers& b,
                const DevGrid& g, const DevPhys& ph) {
#if DEM_ABLATIONS
  if (n <= 0) return K_SWEEP;
  const bool mat = ph.nmat > 1 || ph.nplates > 0;
  const unsigned grid = blocks_for(n, 128);
  if (model == 0) {
    if (mat) k_pair<0, true><<<grid, 128, 0, st>>>(b, g, ph, (uint32_t)n, K);
    else k_pair<0, false><<<grid, 128, 0, st>>>(b, g, ph, (uint32_t)n, K);
  } else {
    if (mat) k_pair<1, true><<<grid, 128, 0, st>>>(b, g, ph, (uint32_t)n, K);
    else k_pair<1, false><<<grid, 128, 0, st>>>(b, g, ph, (uint32_t)n, K);
  }
  // (one warp per 32 owned slots, 4 warps per block)
#endif
  return K_SWEEP;
}

int launch_finish(cudaStream_t st, int64_t n, uint32_t K, int model, bool diag,
                  const StepBuffers& b, const DevGrid& g, const DevPhys& ph) {
#if DEM_ABLATIONS
  if (n <= 0) return K_FINISH;
  const uint32_t N = (uint32_t)n;
  const bool mat = ph.nmat > 1 || ph.nplates > 0;
  const unsigned grid = blocks_for(n, 128);
#define DEM_FIN(M, D)                                                                \
  (mat ? k_finish<M, D, true><<<grid, 128, 0, st>>>(b, g, ph, N, K)                  \
       : k_finish<M, D, false><<<grid, 128, 0, st>>>(b, g, ph, N, K))
  if (model == 0) {
    if (diag) DEM_FIN(0, true);
    else DEM_FIN(0, false);
  } else {
    if (diag) DEM_FIN(1, true);
    else DEM_FIN(1, false);
  }
#undef DEM_FIN
#endif
  return K_FINISH;
}

int launch_detect(cudaStream_t st, int64_t n, uint32_t K, const StepBuffers& b,
                  const DevGrid& g, float mono_r, bool light) {
  if (n <= 0) return K_DETECT;
  constexpr unsigned T = DEM_DETECT_TPB;
  const unsigned grid = blocks_for(n, T);
  if (mono_r > 0.f) {
    const float S = mono_r + mono_r;
    if (light) launch_pdl(k_detect<true, true>, grid, T, 0, st, b, g, (uint32_t)n, K, S * S);
    else launch_pdl(k_detect<true>, grid, T, 0, st, b, g, (uint32_t)n, K, S * S);
  } else {
    if (light) launch_pdl(k_detect<false, true>, grid, T, 0, st, b, g, (uint32_t)n, K, 0.f);
    else launch_pdl(k_detect<false>, grid, T, 0, st, b, g, (uint32_t)n, K, 0.f);
  }
  return K_DETECT;
}

int launch_sweep(cudaStream_t st, int64_t n, uint32_t K, int model, bool diag,
                 const StepBuffers& b, const DevGrid& g, const DevPhys& ph, int variant) {
  if (n <= 0) return K_SWEEP;
  if (model == 0) {
    if (diag)
      sweep_dispatch<0, true>(st, n, K, b, g, ph, variant);
    else
      sweep_dispatch<0, false>(st, n, K, b, g, ph, variant);
  } else {
    if (diag)
      sweep_dispatch<1, true>(st, n, K, b, g, ph, variant);
    else
      sweep_dispatch<1, false>(st, n, K, b, g, ph, variant);
  }
  return K_SWEEP;
}

int launch_plane_hist(cudaStream_t st, int64_t n, const float* pos, DevGrid g, uint32_t* hist) {
  if (n <= 0) return K_OTHER;
  k_plane_hist<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, g, hist);
  return K_OTHER;
}

int launch_keep(cudaStream_t st, int64_t n, const float* pos, DevGrid g, uint32_t* keep) {
  if (n <= 0) return K_OTHER;
  k_keep<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, g, keep);
  return K_OTHER;
}

int launch_flags(cudaStream_t st, int64_t n, const float4* pos, DevGrid g, uint32_t* flags) {
  if (n <= 0) return K_OTHER;
  k_flags<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, g, flags);
  return K_OTHER;
}

// initial = 1: publish the state set by dem_set_particles (xs->n_out preset)
int launch_xpack(cudaStream_t st, int64_t cap, const StepBuffers& b, const DevGrid& g, uint32_t K,
                 uint8_t* mine, XLayout L, XState* xs, int initial, int nbr) {
  const uint32_t ntiles = xtc_ntiles(cap);
  const uint32_t per = L.ghost_cap > L.plane + 1 ? L.ghost_cap : L.plane + 1;
  const unsigned half = (per + 255) / 256;
  if (initial) k_xplanes_initial<<<2 * half, 256, 0, st>>>(b, g, mine, L, nbr);
  else k_xpack_planes<<<2 * half, 256, 0, st>>>(b, g, mine, L, nbr);
  // in a step the integrator has counted the flagged outputs per tile (b.xtc)
  if (initial) k_xpack_count<<<ntiles, 256, 0, st>>>(b, g, b.xtc, ntiles, xs);
  k_xpack_write<<<ntiles, 256, 0, st>>>(b, g, K, (uint32_t)cap, mine, L, b.xtc, b.xtc_next, ntiles,
                                        xs, initial);
  return K_OTHER;
}

int launch_xrecv(cudaStream_t st, int64_t cap, const StepBuffers& b, const DevGrid& g, uint32_t K,
                 const uint8_t* left, const uint8_t* right, XLayout L, XState* xs,
                 uint32_t* nslots_out, bool merge) {
  const uint32_t most = 2 * L.mig_cap + 2 * L.ghost_cap;
  k_xrecv<<<(most + 255) / 256, 256, 0, st>>>(b, g, K, (uint32_t)cap, left, right, L, xs,
                                             nslots_out, merge ? 1 : 0);
  return K_OTHER;
}

int launch_xghost_place(cudaStream_t st, int64_t cap, const StepBuffers& b, const DevGrid& g,
                        const uint8_t* left, const uint8_t* right, XLayout L, XState* xs) {
  const unsigned half = (L.plane + 1 + 255) / 256;
  k_xghost_place<<<2 * half, 256, 0, st>>>(b, g, (uint32_t)cap, left, right, L, xs);
  return K_OTHER;
}

int launch_unpack(cudaStream_t st, int64_t n, bool by_id, const float4* pos, const float4* vel,
                  const float4* omg, const float4* F, const float4* T, float* o_pos,
                  float* o_vel, float* o_omg, float* o_r, float* o_m, uint32_t* o_id,
                  float* o_F, float* o_T, uint32_t idmask, uint32_t* o_mat) {
  if (n <= 0) return K_OTHER;
  k_unpack<<<blocks_for(n, 256), 256, 0, st>>>(n, by_id, pos, vel, omg, F, T, o_pos, o_vel,
                                               o_omg, o_r, o_m, o_id, o_F, o_T, idmask, o_mat);
  return K_OTHER;
}

int launch_emit_contacts(cudaStream_t st, int64_t n, int64_t stride, uint32_t K,
                         const float4* hist, const uint32_t* cnt, const uint32_t* base,
                         const float4* omg, uint32_t* id_i, uint32_t* id_j, float* dt3,
                         uint32_t idmask) {
  if (n <= 0) return K_OTHER;
  k_emit_contacts<<<blocks_for(n, 256), 256, 0, st>>>(n, stride, K, hist, cnt, base, omg, id_i,
                                                      id_j, dt3, idmask);
  return K_OTHER;
}

int launch_slot_of_id(cudaStream_t st, int64_t n, uint32_t idmask, const float4* omg,
                      uint32_t* slot_of_id) {
  if (n <= 0) return K_OTHER;
  k_slot_of_id<<<blocks_for(n, 256), 256, 0, st>>>(n, idmask, omg, slot_of_id);
  return K_OTHER;
}

int launch_insert_contacts(cudaStream_t st, int64_t m, int64_t n, int64_t stride, uint32_t K,
                           const uint32_t* id_i, const uint32_t* id_j, const float* dt3,
                           const uint32_t* slot_of_id, float4* hist, uint32_t* cnt,
                           uint32_t* flags, int skip_unknown) {
  if (m <= 0) return K_OTHER;
  k_insert_contacts<<<blocks_for(m, 256), 256, 0, st>>>(m, n, stride, K, id_i, id_j, dt3,
                                                        slot_of_id, hist, cnt, flags,
                                                        skip_unknown);
  return K_OTHER;
}

int launch_analyze(cudaStream_t st, int64_t n, const StepBuffers& b, const DevGrid& g,
                   unsigned long long* acc) {
  if (n <= 0) return K_OTHER;
  k_analyze<<<blocks_for(n, 256), 256, 0, st>>>(b, g, (uint32_t)n, acc);
  return K_OTHER;
}

int launch_max_speed(cudaStream_t st, int64_t n, const float4* vel, uint32_t* out) {
  if (n <= 0) return K_OTHER;
  k_max_speed<<<296, 256, 0, st>>>(n, vel, out);
  return K_OTHER;
}

int launch_cnt_stats(cudaStream_t st, int64_t n, const uint32_t* cnt,
                     unsigned long long* sum_max) {
  if (n <= 0) return K_OTHER;
  k_cnt_stats<<<296, 256, 0, st>>>(n, cnt, sum_max);
  return K_OTHER;
}

}  // namespace dem

// rk_tsdf.cu -- K4 block activation over a GPU open-addressing hash, K5
// voxel-parallel projective TSDF integration, block I/O and trilinear queries.
//
// Storage: a pool of 16^3 blocks, each 4096 float2
// {tsdf, weight} voxels in C order (z fastest) = 32 KB, addressed by slot.
// Keys are packed exactly like sdf_volume.py:64-71 (bias 2^17, 2^18 per axis)
// into a 64-bit word; the hash maps key -> slot with linear probing.  Each
// activation appends the frame's touched hash entries to a list (deduplicated
// by a per-entry frame stamp) -- the touched set the reference returns.
#include "rk_common.cuh"

using namespace rk;

// K5 launch shape: RK_TSDF_THREADS x RK_TSDF_CTAS_PER_SM persistent CTAs per SM
#ifndef RK_TSDF_THREADS
#define RK_TSDF_THREADS 256
#endif
#ifndef RK_TSDF_CTAS_PER_SM
#define RK_TSDF_CTAS_PER_SM 4  // 62 registers, no spills; +3% over 3 CTAs/SM (which left room for the side-stream activation)
#endif

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

namespace {

constexpr int kEdge = 16;
constexpr int kVox = kEdge * kEdge * kEdge;
constexpr long long kBias = 1ll << 17;
constexpr long long kShift = 1ll << 18;
constexpr unsigned long long kEmpty = ~0ull;
constexpr int kChunkBlocks = 600000 / kVox;  // sdf_volume.py:142 (146 blocks)

// per-frame touched set bookkeeping; two slots so that the activation of
// frame f+1 can run while frame f integrates (rk_grid_integrate_frames)
struct TouchCounters {
  unsigned long long max_touched_key;  // largest packed key touched this frame
  long long n_touched;
};

struct Counters {
  long long n_blocks;                  // allocated slots
  long long updated;                   // voxels updated by the last integrate
  int n_fresh;
  int overflow;
  int n_points;                        // activation input size (gemv quirk)
  int frame;                           // activation stamp (device-side: graph-replay safe)
  int work;                            // k_integrate's dynamic block counter
  int done;                            // k_integrate's finished-CTA ticket
};

__host__ __device__ __forceinline__ unsigned long long pack_key(long long x, long long y, long long z) {
  return (unsigned long long)(((x + kBias) * kShift + (y + kBias)) * kShift + (z + kBias));
}
__host__ __device__ __forceinline__ void unpack_key(unsigned long long p, int& x, int& y, int& z) {
  long long q = (long long)p;
  z = (int)(q % kShift - kBias);
  q /= kShift;
  y = (int)(q % kShift - kBias);
  x = (int)(q / kShift - kBias);
}
__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

struct GridDev {
  float2* vox;
  int4* block_keys;
  unsigned long long* h_keys;
  int32_t* h_slot;
  int32_t* h_stamp;
  int32_t* touched;      // this view's touched list (slot base + slot * hash capacity)
  int32_t* fresh;
  Counters* ctr;
  TouchCounters* tc;     // this view's touched counters
  long long cap_blocks;
  unsigned long long hash_mask;
  int shard_rank, shard_world;  // multi-GPU: this grid keeps owner(key) == rank
};

// find or insert; returns hash position or -1 when the probe budget is spent
__device__ long long hash_acquire(const GridDev& g, unsigned long long key, bool& inserted) {
  unsigned long long h = mix64(key) & g.hash_mask;
  inserted = false;
  for (int probe = 0; probe < 4096; ++probe) {
    unsigned long long k = *((volatile unsigned long long*)(g.h_keys + h));
    if (k == key) return (long long)h;
    if (k == kEmpty) {
      unsigned long long prev = atomicCAS(g.h_keys + h, kEmpty, key);
      if (prev == kEmpty) { inserted = true; return (long long)h; }
      if (prev == key) return (long long)h;
    }
    h = (h + 1) & g.hash_mask;
  }
  return -1;
}

__device__ long long hash_find(const GridDev& g, unsigned long long key) {
  unsigned long long h = mix64(key) & g.hash_mask;
  for (int probe = 0; probe < 4096; ++probe) {
    unsigned long long k = g.h_keys[h];
    if (k == key) return (long long)h;
    if (k == kEmpty) return -1;
    h = (h + 1) & g.hash_mask;
  }
  return -1;
}

// one touched key: insert, dedupe per frame, remember fresh keys
__device__ __forceinline__ void touch_key(const GridDev& g, int frame, long long x, long long y, long long z) {
  unsigned long long key = pack_key(x, y, z);
  if (g.shard_world > 1 && (int)(rk_owner_mix(key) % (unsigned long long)g.shard_world) != g.shard_rank)
    return;  // another GPU owns this block
  bool inserted;
  long long h = hash_acquire(g, key, inserted);
  if (h < 0) { atomicExch(&g.ctr->overflow, 1); return; }
  RK_DCHECK((unsigned long long)h <= g.hash_mask, "K4 hash slot", h, g.hash_mask);
  if (inserted) {
    const int fi = atomicAdd(&g.ctr->n_fresh, 1);
    RK_DCHECK((unsigned long long)fi <= g.hash_mask, "K4 fresh list", fi, g.hash_mask);
    g.fresh[fi] = (int32_t)h;
  }
  if (g.h_stamp[h] != frame && atomicExch(g.h_stamp + h, frame) != frame) {
    const unsigned long long ti = atomicAdd(reinterpret_cast<unsigned long long*>(&g.tc->n_touched), 1ull);
    RK_DCHECK(ti <= g.hash_mask, "K4 touched list", ti, g.hash_mask);
    g.touched[ti] = (int32_t)h;
    atomicMax(&g.tc->max_touched_key, key);
  }
}

// all keys of blocks meeting the cube [p - radius, p + radius] (sdf_volume.py:88-106)
__device__ __forceinline__ void touch_point(const GridDev& g, int frame, const double p[3],
                                            double radius, double ext) {
  long long lo[3], hi[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = (long long)floor(__ddiv_rn(__dsub_rn(p[c], radius), ext));
    hi[c] = (long long)floor(__ddiv_rn(__dadd_rn(p[c], radius), ext));
  }
  for (long long x = lo[0]; x <= hi[0]; ++x)
    for (long long y = lo[1]; y <= hi[1]; ++y)
      for (long long z = lo[2]; z <= hi[2]; ++z) touch_key(g, frame, x, y, z);
}

__device__ __forceinline__ void reset_frame(Counters* c, TouchCounters* t) {
  c->frame += 1;
  c->n_fresh = 0;
  t->n_touched = 0;
  t->max_touched_key = 0ull;
}
__global__ void k_reset_frame(Counters* c, TouchCounters* t) { reset_frame(c, t); }

// touch_point for a whole warp.  A warp is 32 neighbouring pixels of one
// row, so its cubes share few block keys: lanes elect one lane per distinct
// key (__match_any_sync) into a per-warp list in shared memory, then the warp
// resolves the list's keys in parallel -- one round of dependent hash/stamp
// atomics per warp instead of up to 8 per point.  Every lane must call it;
// `list` holds 32 * max-keys-per-point entries.
constexpr int kMaxKeysPerPoint = 8;
__device__ __forceinline__ void touch_point_warp(const GridDev& g, int frame, const double p[3],
                                                 bool valid, double radius, double ext,
                                                 unsigned long long* list) {
  long long lo[3] = {0, 0, 0};
  int n[3] = {0, 0, 0};
  if (valid) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = (long long)floor(__ddiv_rn(__dsub_rn(p[c], radius), ext));
      const long long hi = (long long)floor(__ddiv_rn(__dadd_rn(p[c], radius), ext));
      n[c] = (int)(hi - lo[c] + 1);
    }
  }
  const int total = n[0] * n[1] * n[2];
  const int lane = threadIdx.x & 31;
  const int rounds = __reduce_max_sync(0xffffffffu, total);
  int n_list = 0;
  for (int j = 0; j < rounds; ++j) {
    unsigned long long key = kEmpty;
    if (j < total) {
      const int iz = j % n[2], iy = (j / n[2]) % n[1], ix = j / (n[2] * n[1]);
      key = pack_key(lo[0] + ix, lo[1] + iy, lo[2] + iz);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const bool lead = key != kEmpty && lane == __ffs(peers) - 1;
    const unsigned leaders = __ballot_sync(0xffffffffu, lead);
    if (lead && n_list + __popc(leaders & ((1u << lane) - 1u)) < 32 * kMaxKeysPerPoint)
      list[n_list + __popc(leaders & ((1u << lane) - 1u))] = key;
    n_list = min(n_list + __popc(leaders), 32 * kMaxKeysPerPoint);
    if (n_list == 32 * kMaxKeysPerPoint || j + 1 == rounds) {  // flush (duplicates across rounds are harmless)
      __syncwarp();
      for (int t = lane; t < n_list; t += 32) {
        int x, y, z;
        unpack_key(list[t], x, y, z);
        touch_key(g, frame, x, y, z);
      }
      __syncwarp();
      n_list = 0;
    }
  }
}

__global__ void k_activate_points(GridDev g, const double* __restrict__ pts, int64_t n,
                                  double radius, double ext) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int frame = g.ctr->frame;
  double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  touch_point(g, frame, p, radius, ext);
}

// open a new frame (stamp, counters; CTA 0) and count the frame's valid
// pixels (to_point_cloud size, needed for the single-row gemv quirk) into
// n_points, which the previous k_assign_slots left at zero
constexpr int kBeginThreads = 256, kBeginCtas = 64;
__global__ void __launch_bounds__(kBeginThreads) k_begin_image_frame(const float* __restrict__ range, int n,
                                                                      float cmin, float cmax, Counters* c,
                                                                      TouchCounters* t) {
  __shared__ int part[kBeginThreads / 32];
  if (blockIdx.x == 0 && threadIdx.x == 0) reset_frame(c, t);
  int cnt = 0;
  for (int i = blockIdx.x * kBeginThreads + threadIdx.x; i < n; i += kBeginThreads * gridDim.x)
    cnt += range_ok(__ldg(range + i), cmin, cmax) ? 1 : 0;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kBeginThreads / 32; ++w) tot += part[w];
    if (tot) atomicAdd(&c->n_points, tot);
  }
}

// to_point_cloud -> pose.apply -> activate_blocks, fused (sdf_volume.py:198-208)
__global__ void __launch_bounds__(256) k_activate_image(GridDev g, SensorDev s, const float* __restrict__ range,
                                 const double* __restrict__ pose12, double radius, double ext,
                                 float cmin, float cmax) {
  __shared__ unsigned long long keys[256 / 32][32 * kMaxKeysPerPoint];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // whole warps stay (warp dedup)
  const int frame = g.ctr->frame;
  const bool in = i < s.H * s.W;
  const float r = in ? range[i] : 0.0f;
  const bool valid = in && range_ok(r, cmin, cmax);
  double w[3] = {0.0, 0.0, 0.0};
  if (valid) {
    double pose[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) pose[k] = pose12[k];
    double p[3];
    unproject_px(s, i / s.W, i % s.W, r, p);
    xform_rows(pose, pose + 9, p[0], p[1], p[2], w, g.ctr->n_points == 1);
  }
  touch_point_warp(g, frame, w, valid, radius, ext, keys[threadIdx.x >> 5]);
}

// fresh keys -> pool slots (slot order follows the fresh list); one CTA,
// which then publishes the new block count
constexpr int kAssignThreads = 1024;
__global__ void __launch_bounds__(kAssignThreads) k_assign_slots(GridDev g) {
  const int nf = g.ctr->n_fresh;
  const long long base = g.ctr->n_blocks;
  for (int i = threadIdx.x; i < nf; i += kAssignThreads) {
    int h = g.fresh[i];
    long long slot = base + i;
    if (slot < g.cap_blocks) {
      g.h_slot[h] = (int32_t)slot;
      int x, y, z;
      unpack_key(g.h_keys[h], x, y, z);
      g.block_keys[slot] = make_int4(x, y, z, 0);
    } else {
      g.h_slot[h] = -1;
      atomicExch(&g.ctr->overflow, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long nb = base + nf;
    g.ctr->n_blocks = nb < g.cap_blocks ? nb : g.cap_blocks;
    g.ctr->n_fresh = 0;
    g.ctr->n_points = 0;  // k_begin_image_frame of the next frame accumulates into it
  }
}

#ifndef RK_TSDF_FAST_PROJ
#define RK_TSDF_FAST_PROJ 1
#endif
#ifndef RK_TSDF_STATIC
#define RK_TSDF_STATIC 1
#endif
#ifndef RK_TSDF_EARLY_STATE
#define RK_TSDF_EARLY_STATE 1
#endif
#ifndef RK_TSDF_PREFETCH  // +2.6% at C5 (grid in HBM), +-0 at C2 (A/B r2x)
#define RK_TSDF_PREFETCH 1
#endif
// RK_TSDF_STATE_HINT: stream the voxel states with the evict-first
// (cache-streaming) policy, ld.global.cs / st.global.cs, so a grid larger
// than L2 does not push the range image and the row tables out of it
#ifndef RK_TSDF_STATE_HINT  // with the prefetch: +2.9% at C5, +-0 at C2 (A/B r2x)
#define RK_TSDF_STATE_HINT 1
#endif
__device__ __forceinline__ float2 load_state(const float2* p) {
#if RK_TSDF_STATE_HINT
  return __ldcs(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void store_state(float2* p, float2 v) {
#if RK_TSDF_STATE_HINT
  __stcs(p, v);
#else
  *p = v;
#endif
}
#ifndef RK_TSDF_UNROLL
#define RK_TSDF_UNROLL 8  // voxel-loop unroll of k_integrate: 8 beat 2 by +1.8% TSDF fps (A/B x3, r1o); 1 -1.3%, 4 +1.2%, 16 -1.6%; no spills
#endif
constexpr int kIntegrateUnroll = RK_TSDF_UNROLL;

// bulk L2 prefetch of one block's voxel states (TMA unit, no registers held)
__device__ __forceinline__ void prefetch_block_l2(const float2* p) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)(kVox * sizeof(float2)))
               : "memory");
}

struct IntegrateArgs {
  GridDev g;
  SensorDev s;
  const float* range;
  const double* inv12;
  double voxel;
  double block_ext;  // 16 * voxel_size
  float tau, max_w, cmin, cmax;
  int free_space;
  long long* updated;
  const long long* global_touch;  // sharded grids: {frame key count, max key} over all ranks
};

// K5: persistent CTAs (kIntegrateCtasPerSm per SM) pull touched blocks from
// a device counter; each block's 4096 voxels are projected into the
// (L2-resident) range image and folded into the running average; voxels whose
// observation is rejected cost no state traffic.  Every CTA first builds the
// frame's rotated voxel-centre lattice in shared memory (sdf_volume.py:160:
// f32(((local + 0.5) * voxel) @ inv.R^T), the OpenBLAS FMA order) -- 36
// float64 ops per thread instead of a separate launch and a 48 KB copy.
template <int MATH, int NT, bool SMEM>
__global__ void __launch_bounds__(NT, RK_TSDF_CTAS_PER_SM) k_integrate(IntegrateArgs A) {
  extern __shared__ float sh_off[];  // kVox*3 rotated lattice (48 KB, dynamic)
  __shared__ int sh_cnt[NT / 32];
#if !RK_TSDF_STATIC
  __shared__ int sh_e;
#endif
  __shared__ RowTablesSmem sh_tab;
#if RK_TSDF_STATIC && RK_TSDF_PREFETCH
  // the first block's states stream into L2 while the lattice is built
  if (threadIdx.x == 0 && blockIdx.x < (int)A.g.tc->n_touched) {
    const int s0 = A.g.h_slot[A.g.touched[blockIdx.x]];
    if (s0 >= 0) prefetch_block_l2(A.g.vox + (size_t)s0 * kVox);
  }
#endif
  if (SMEM) stage_tables(A.s, sh_tab, threadIdx.x, NT);
  const RowTables tb = SMEM ? RowTables{sh_tab.el32, sh_tab.az32, sh_tab.inv_rows} : global_tables(A.s);
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = A.inv12[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = A.inv12[9 + k];
  for (int i = threadIdx.x; i < kVox; i += NT) {
    const double l0 = __dmul_rn(__dadd_rn((double)(i >> 8), 0.5), A.voxel);
    const double l1 = __dmul_rn(__dadd_rn((double)((i >> 4) & 15), 0.5), A.voxel);
    const double l2 = __dmul_rn(__dadd_rn((double)(i & 15), 0.5), A.voxel);
    double o[3];
    xform_rows(R, nullptr, l0, l1, l2, o);
    sh_off[3 * i] = (float)o[0];
    sh_off[3 * i + 1] = (float)o[1];
    sh_off[3 * i + 2] = (float)o[2];
  }
  __syncthreads();
  const SensorDev& s = A.s;
  const int n_touched = (int)A.g.tc->n_touched;
  // the reference integrates sorted keys in chunks of 146 blocks; a chunk of a
  // single block goes through dgemv, which orders the FMA chain differently.
  // A hash-sharded grid needs the frame's global count / largest key, which
  // the caller all-reduces into global_touch = {count, max key}.
  const long long n_all = A.global_touch ? A.global_touch[0] : n_touched;
  const unsigned long long max_key =
      A.global_touch ? (unsigned long long)A.global_touch[1] : A.g.tc->max_touched_key;
  const bool lone_tail = (n_all % kChunkBlocks) == 1;
  int count = 0;
#if RK_TSDF_STATIC
  // static round-robin blocks: the next block is known, so its metadata
  // (touched entry -> slot, key) is loaded while the current one runs
  int h_n = blockIdx.x < n_touched ? A.g.touched[blockIdx.x] : 0;
  int slot_n = blockIdx.x < n_touched ? A.g.h_slot[h_n] : -1;
  unsigned long long key_n = blockIdx.x < n_touched ? A.g.h_keys[h_n] : 0ull;
  for (int e = blockIdx.x; e < n_touched; e += gridDim.x) {
    const int slot = slot_n;
    const unsigned long long key = key_n;
    const int e2 = e + gridDim.x;
    if (e2 < n_touched) {
      h_n = A.g.touched[e2];
      slot_n = A.g.h_slot[h_n];
      key_n = A.g.h_keys[h_n];
#if RK_TSDF_PREFETCH
      // the next block's states stream into L2 while this block runs
      if (threadIdx.x == 0 && slot_n >= 0) prefetch_block_l2(A.g.vox + (size_t)slot_n * kVox);
#endif
    }
    if (slot < 0) continue;
#else
  for (;;) {
    if (threadIdx.x == 0) sh_e = atomicAdd(&A.g.ctr->work, 1);
    __syncthreads();
    const int e = sh_e;
    __syncthreads();  // sh_e is rewritten by the next fetch
    if (e >= n_touched) break;
    const int h = A.g.touched[e];
    const int slot = A.g.h_slot[h];
    if (slot < 0) continue;
    const unsigned long long key = A.g.h_keys[h];
#endif
    RK_DCHECK(slot < A.g.cap_blocks, "K5 voxel slot", slot, A.g.cap_blocks);
    int kx, ky, kz;
    unpack_key(key, kx, ky, kz);
    double base[3];
    xform_rows(R, t, __dmul_rn((double)kx, A.block_ext), __dmul_rn((double)ky, A.block_ext),
               __dmul_rn((double)kz, A.block_ext), base, lone_tail && key == max_key);
    const float bx = (float)base[0], by = (float)base[1], bz = (float)base[2];
    float2* vox = A.g.vox + (size_t)slot * kVox;
#pragma unroll kIntegrateUnroll
    for (int i = threadIdx.x; i < kVox; i += NT) {
#if RK_TSDF_EARLY_STATE
      // the voxel state does not depend on the observation: issue its load
      // first so the projection math hides the latency
      float2 st0 = load_state(vox + i);
#endif
      const float x = __fadd_rn(bx, sh_off[3 * i]);
      const float y = __fadd_rn(by, sh_off[3 * i + 1]);
      const float z = __fadd_rn(bz, sh_off[3 * i + 2]);
      Proj32 p = project_f32<MATH, SMEM, MATH != MATH_FAST ? PROJ_EXACT_FINITE : RK_TSDF_FAST_PROJ ? PROJ_FAST_R : PROJ_EXACT>(s, tb, x, y, z);
      int col = (int)__fadd_rn(p.u, 0.5f);
      if (col == s.W) col = 0;
      RK_DCHECK(p.v >= 0 && p.v < s.H && col >= 0 && col < s.W, "K5 range gather", p.v, col);
      const int pix = p.v * s.W + col;  // one 32-bit index: a single wide IMAD for the address
      const float px = __ldg(A.range + pix);
      bool ok = p.status == PROJ_OK && px > 0.0f && px >= A.cmin && px <= A.cmax && p.r <= A.cmax;
      float d = __fsub_rn(px, p.r);
      ok = ok && d >= -A.tau;
      if (!A.free_space) ok = ok && d <= A.tau;
      d = fminf(d, A.tau);
      if (ok) {
#if RK_TSDF_EARLY_STATE
        float2 st = st0;
#else
        float2 st = load_state(vox + i);
#endif
        const float wn = __fadd_rn(st.y, 1.0f);
        // (w*tsdf + d) / (w + 1), correctly rounded (w + 1 in [1, max_weight + 1])
        st.x = MATH != MATH_CR ? div_rn_fast(__fadd_rn(__fmul_rn(st.y, st.x), d), wn)
                               : __fdiv_rn(__fadd_rn(__fmul_rn(st.y, st.x), d), wn);
        st.y = fminf(wn, A.max_w);
        store_state(vox + i, st);
        ++count;
      }
    }
  }
  count = __reduce_add_sync(0xffffffffu, count);
  if ((threadIdx.x & 31) == 0) sh_cnt[threadIdx.x >> 5] = count;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (A.updated) {
      long long tot = 0;
      for (int w = 0; w < NT / 32; ++w) tot += sh_cnt[w];
      if (tot) atomicAdd((unsigned long long*)A.updated, (unsigned long long)tot);
    }
    // the last CTA out rewinds the block counter for the next launch (every
    // CTA has stopped fetching once it takes its ticket)
    __threadfence();
    if (atomicAdd(&A.g.ctr->done, 1) == (int)gridDim.x - 1) {
      A.g.ctr->work = 0;
      A.g.ctr->done = 0;
    }
  }
}

__global__ void k_set_touched(GridDev g, const int32_t* __restrict__ keys, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int frame = g.ctr->frame;
  // explicit frame_keys: they need not exist yet (integrate() on unknown keys
  // raises KeyError in the reference; here they are simply skipped)
  unsigned long long key = pack_key(keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]);
  long long h = hash_find(g, key);
  if (h < 0) return;
  if (atomicExch(g.h_stamp + h, frame) != frame) {
    g.touched[atomicAdd(reinterpret_cast<unsigned long long*>(&g.tc->n_touched), 1ull)] = (int32_t)h;
    atomicMax(&g.tc->max_touched_key, key);
  }
}

__global__ void k_keys_all(GridDev g, int32_t* out, long long cap) {
  long long nb = g.ctr->n_blocks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nb && i < cap;
       i += (long long)gridDim.x * blockDim.x) {
    int4 k = g.block_keys[i];
    out[3 * i] = k.x;
    out[3 * i + 1] = k.y;
    out[3 * i + 2] = k.z;
  }
}

__global__ void k_keys_touched(GridDev g, int32_t* out, long long cap) {
  const long long nt = g.tc->n_touched;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nt && i < cap;
       i += (long long)gridDim.x * blockDim.x) {
    int x, y, z;
    unpack_key(g.h_keys[g.touched[i]], x, y, z);
    out[3 * i] = x;
    out[3 * i + 1] = y;
    out[3 * i + 2] = z;
  }
}

__global__ void k_read_blocks(GridDev g, const int32_t* __restrict__ keys, int64_t n, float2* out,
                              uint8_t* found) {
  int64_t b = blockIdx.x;
  if (b >= n) return;
  long long h = hash_find(g, pack_key(keys[3 * b], keys[3 * b + 1], keys[3 * b + 2]));
  int slot = h >= 0 ? g.h_slot[h] : -1;
  if (threadIdx.x == 0 && found) found[b] = slot >= 0;
  float2* dst = out + b * kVox;
  if (slot < 0) {
    for (int i = threadIdx.x; i < kVox; i += blockDim.x) dst[i] = make_float2(0.f, 0.f);
    return;
  }
  const float2* src = g.vox + (size_t)slot * kVox;
  for (int i = threadIdx.x; i < kVox; i += blockDim.x) dst[i] = src[i];
}

__global__ void k_insert_keys(GridDev g, const int32_t* __restrict__ keys, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool inserted;
  long long h = hash_acquire(g, pack_key(keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]), inserted);
  if (h < 0) { atomicExch(&g.ctr->overflow, 1); return; }
  if (inserted) g.fresh[atomicAdd(&g.ctr->n_fresh, 1)] = (int32_t)h;
}

__global__ void k_write_blocks(GridDev g, const int32_t* __restrict__ keys, int64_t n, const float2* src) {
  int64_t b = blockIdx.x;
  if (b >= n) return;
  long long h = hash_find(g, pack_key(keys[3 * b], keys[3 * b + 1], keys[3 * b + 2]));
  int slot = h >= 0 ? g.h_slot[h] : -1;
  if (slot < 0) return;
  float2* dst = g.vox + (size_t)slot * kVox;
  for (int i = threadIdx.x; i < kVox; i += blockDim.x) dst[i] = src[b * kVox + i];
}

__device__ __forceinline__ void voxel_at(const GridDev& g, long long gx, long long gy, long long gz,
                                         float& d, float& w, bool& found) {
  long long bx = gx >= 0 ? gx / kEdge : -((-gx + kEdge - 1) / kEdge);
  long long by = gy >= 0 ? gy / kEdge : -((-gy + kEdge - 1) / kEdge);
  long long bz = gz >= 0 ? gz / kEdge : -((-gz + kEdge - 1) / kEdge);
  long long h = hash_find(g, pack_key(bx, by, bz));
  int slot = h >= 0 ? g.h_slot[h] : -1;
  found = slot >= 0;
  d = w = 0.f;
  if (!found) return;
  int lx = (int)(gx - bx * kEdge), ly = (int)(gy - by * kEdge), lz = (int)(gz - bz * kEdge);
  float2 v = g.vox[(size_t)slot * kVox + (lx * kEdge + ly) * kEdge + lz];
  d = v.x;
  w = v.y;
}

// query_sdf_many (sdf_volume.py:221-244): trilinear over the 8 enclosing centres
__global__ void k_query(GridDev g, double voxel, const double* __restrict__ pts, int64_t n,
                        double* sdf, double* wt, uint8_t* obs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double gq[3], fr[3];
  long long b[3];
  for (int c = 0; c < 3; ++c) {
    gq[c] = __dsub_rn(__ddiv_rn(pts[3 * i + c], voxel), 0.5);
    double f = floor(gq[c]);
    b[c] = (long long)f;
    fr[c] = __dsub_rn(gq[c], (double)b[c]);
  }
  double s_acc = 0.0, w_acc = 0.0;
  bool ok = true;
  for (int corner = 0; corner < 8; ++corner) {
    int cx = (corner >> 2) & 1, cy = (corner >> 1) & 1, cz = corner & 1;
    double w0 = cx ? fr[0] : __dsub_rn(1.0, fr[0]);
    double w1 = cy ? fr[1] : __dsub_rn(1.0, fr[1]);
    double w2 = cz ? fr[2] : __dsub_rn(1.0, fr[2]);
    double cw = __dmul_rn(__dmul_rn(w0, w1), w2);
    float d, w;
    bool found;
    voxel_at(g, b[0] + cx, b[1] + cy, b[2] + cz, d, w, found);
    ok = ok && found && w > 0.f;
    s_acc = __dadd_rn(s_acc, __dmul_rn(cw, (double)d));
    w_acc = __dadd_rn(w_acc, __dmul_rn(cw, (double)w));
  }
  sdf[i] = s_acc;
  wt[i] = w_acc;
  obs[i] = ok ? 1 : 0;
}

__global__ void k_rehash(GridDev g, long long nb) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nb;
       i += (long long)gridDim.x * blockDim.x) {
    int4 k = g.block_keys[i];
    bool inserted;
    long long h = hash_acquire(g, pack_key(k.x, k.y, k.z), inserted);
    if (h >= 0) g.h_slot[h] = (int32_t)i;
  }
}

}  // namespace

// ------------------------------------------------------------------ host side
constexpr int kIntegrateThreads = RK_TSDF_THREADS;
constexpr int kIntegrateCtasPerSm = RK_TSDF_CTAS_PER_SM;
constexpr size_t kLatticeBytes = kVox * 3 * sizeof(float);

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static cudaError_t set_integrate_attrs() {
  constexpr int NT = kIntegrateThreads;
  (void)num_sms();  // cached now: rk_grid_integrate may later run under graph capture
  const int smem = (int)kLatticeBytes;
  cudaError_t e;
  const void* fns[] = {(const void*)k_integrate<MATH_CR, NT, true>, (const void*)k_integrate<MATH_CR, NT, false>,
                       (const void*)k_integrate<MATH_FAST, NT, true>, (const void*)k_integrate<MATH_FAST, NT, false>,
                       (const void*)k_integrate<MATH_NP, NT, true>, (const void*)k_integrate<MATH_NP, NT, false>};
  for (const void* f : fns)
    if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  return cudaSuccess;
}

struct rk_grid {
  double voxel, trunc;
  float max_weight;
  int free_space;
  GridDev d;              // slot-0 view; d.touched / d.tc are the bases of both slots
  unsigned long long hash_cap;
  int last_slot = 0;      // touched-set slot of the most recent activation
  int n_slots = 2;        // touched-set slots (>= 2; rk_grid_reserve_slots grows them)
  const long long* global_touch = nullptr;  // device {count, max key} (sharded grids)
  cudaStream_t side = nullptr;               // activation stream of rk_grid_integrate_frames
  cudaEvent_t ev_act[2] = {nullptr, nullptr}, ev_int[2] = {nullptr, nullptr}, ev_fork = nullptr;
  void* scratch[2] = {nullptr, nullptr};     // rk_grid_scratch_ (marching cubes output)
  size_t scratch_bytes[2] = {0, 0};
};

void* rk_grid_scratch_(rk_grid* g, int which, size_t bytes) {
  if (bytes > g->scratch_bytes[which]) {
    if (g->scratch[which]) {
      cudaDeviceSynchronize();  // earlier users of the slot may still be running
      cudaFree(g->scratch[which]);
      g->scratch[which] = nullptr;
      g->scratch_bytes[which] = 0;
    }
    const size_t want = bytes + bytes / 4;  // headroom: meshes grow with the grid
    cudaError_t e = cudaMalloc(&g->scratch[which], want);
    if (e != cudaSuccess) {
      rk_cuda_status(e, "rk_grid_scratch_");
      return nullptr;
    }
    g->scratch_bytes[which] = want;
  }
  return g->scratch[which];
}

// the grid as seen by the kernels of one touched-set slot
static GridDev view(const rk_grid* g, int slot) {
  GridDev v = g->d;
  v.touched = g->d.touched + (size_t)slot * g->hash_cap;
  v.tc = g->d.tc + slot;
  return v;
}

// {n_touched, max touched key} of the last activation into a device int64[2]
// (multi-GPU: all-reduce these with sum / max, then rk_grid_set_global_touch)
__global__ void k_touch_stats(const TouchCounters* t, long long* out) {
  out[0] = t->n_touched;
  out[1] = (long long)t->max_touched_key;
}

extern "C" int rk_grid_touch_stats(rk_grid* g, int64_t* out2, void* stream) {
  k_touch_stats<<<1, 1, 0, S(stream)>>>(g->d.tc + g->last_slot, reinterpret_cast<long long*>(out2));
  RK_LAUNCHED("k_touch_stats");
  return RK_OK;
}

extern "C" int rk_grid_set_global_touch(rk_grid* g, const int64_t* in2) {
  g->global_touch = reinterpret_cast<const long long*>(in2);
  return RK_OK;
}

static unsigned long long pow2_at_least(unsigned long long x) {
  unsigned long long p = 1024;
  while (p < x) p <<= 1;
  return p;
}

static int alloc_tables(rk_grid* g, long long cap_blocks, cudaStream_t st) {
  GridDev& d = g->d;
  unsigned long long hcap = pow2_at_least((unsigned long long)cap_blocks * 4ull);
  RK_CUDA(cudaMalloc(&d.vox, (size_t)cap_blocks * kVox * sizeof(float2)));
  RK_CUDA(cudaMemsetAsync(d.vox, 0, (size_t)cap_blocks * kVox * sizeof(float2), st));
  RK_CUDA(cudaMalloc(&d.block_keys, (size_t)cap_blocks * sizeof(int4)));
  RK_CUDA(cudaMalloc(&d.h_keys, hcap * sizeof(unsigned long long)));
  RK_CUDA(cudaMemsetAsync(d.h_keys, 0xff, hcap * sizeof(unsigned long long), st));
  RK_CUDA(cudaMalloc(&d.h_slot, hcap * sizeof(int32_t)));
  RK_CUDA(cudaMemsetAsync(d.h_slot, 0xff, hcap * sizeof(int32_t), st));
  RK_CUDA(cudaMalloc(&d.h_stamp, hcap * sizeof(int32_t)));
  RK_CUDA(cudaMemsetAsync(d.h_stamp, 0, hcap * sizeof(int32_t), st));
  RK_CUDA(cudaMalloc(&d.touched, (size_t)g->n_slots * hcap * sizeof(int32_t)));  // touched-set slots
  RK_CUDA(cudaMalloc(&d.fresh, hcap * sizeof(int32_t)));
  d.cap_blocks = cap_blocks;
  d.hash_mask = hcap - 1;
  g->hash_cap = hcap;
  return RK_OK;
}

static void free_tables(GridDev& d) {
  cudaFree(d.vox);
  cudaFree(d.block_keys);
  cudaFree(d.h_keys);
  cudaFree(d.h_slot);
  cudaFree(d.h_stamp);
  cudaFree(d.touched);
  cudaFree(d.fresh);
}

extern "C" int rk_grid_create(double voxel_size, double truncation, float max_weight,
                              int32_t free_space, int64_t capacity_blocks, rk_grid** out) {
  if (!(voxel_size > 0) || !(truncation > 0)) {
    rk_set_error("voxel size and truncation must be > 0");
    return RK_EGENERIC;
  }
  rk_grid* g = new rk_grid();
  g->voxel = voxel_size;
  g->trunc = truncation;
  g->max_weight = max_weight;
  g->free_space = free_space;
  g->d.shard_rank = 0;
  g->d.shard_world = 1;
  if (capacity_blocks < 64) capacity_blocks = 64;
  int rc = alloc_tables(g, capacity_blocks, 0);
  if (rc) { delete g; return rc; }
  RK_CUDA(cudaMalloc(&g->d.ctr, sizeof(Counters)));
  RK_CUDA(cudaMemset(g->d.ctr, 0, sizeof(Counters)));
  RK_CUDA(cudaMalloc(&g->d.tc, g->n_slots * sizeof(TouchCounters)));
  RK_CUDA(cudaMemset(g->d.tc, 0, g->n_slots * sizeof(TouchCounters)));
  RK_CUDA(set_integrate_attrs());
  // side stream + events of rk_grid_integrate_frames, created here so that the
  // sequence call itself can run under stream capture
  RK_CUDA(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    RK_CUDA(cudaEventCreateWithFlags(&g->ev_act[i], cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&g->ev_int[i], cudaEventDisableTiming));
  }
  RK_CUDA(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
  RK_CUDA(cudaDeviceSynchronize());
  *out = g;
  return RK_OK;
}

extern "C" int rk_grid_destroy(rk_grid* g) {
  if (!g) return RK_OK;
  cudaDeviceSynchronize();
  free_tables(g->d);
  cudaFree(g->d.ctr);
  cudaFree(g->d.tc);
  cudaFree(g->scratch[0]);
  cudaFree(g->scratch[1]);
  if (g->side) {
    cudaStreamDestroy(g->side);
    for (int i = 0; i < 2; ++i) { cudaEventDestroy(g->ev_act[i]); cudaEventDestroy(g->ev_int[i]); }
    cudaEventDestroy(g->ev_fork);
  }
  delete g;
  return RK_OK;
}

extern "C" int rk_grid_reserve(rk_grid* g, int64_t capacity_blocks, void* stream) {
  cudaStream_t st = S(stream);
  if (capacity_blocks <= g->d.cap_blocks) return RK_OK;
  Counters c;
  RK_CUDA(cudaMemcpyAsync(&c, g->d.ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  GridDev old = g->d;
  int rc = alloc_tables(g, capacity_blocks, st);
  if (rc) return rc;
  long long nb = c.n_blocks;
  if (nb > 0) {
    RK_CUDA(cudaMemcpyAsync(g->d.vox, old.vox, (size_t)nb * kVox * sizeof(float2),
                            cudaMemcpyDeviceToDevice, st));
    RK_CUDA(cudaMemcpyAsync(g->d.block_keys, old.block_keys, (size_t)nb * sizeof(int4),
                            cudaMemcpyDeviceToDevice, st));
    k_rehash<<<256, 256, 0, st>>>(g->d, nb);
    RK_LAUNCHED("k_rehash");
  }
  c.overflow = 0;
  c.n_fresh = 0;
  RK_CUDA(cudaMemcpyAsync(g->d.ctr, &c, sizeof(c), cudaMemcpyHostToDevice, st));
  RK_CUDA(cudaMemsetAsync(g->d.tc, 0, g->n_slots * sizeof(TouchCounters), st));
  RK_CUDA(cudaStreamSynchronize(st));
  free_tables(old);
  return RK_OK;
}

extern "C" int rk_grid_info(rk_grid* g, int64_t* out4, void* stream) {
  cudaStream_t st = S(stream);
  Counters c;
  TouchCounters t;
  RK_CUDA(cudaMemcpyAsync(&c, g->d.ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaMemcpyAsync(&t, g->d.tc + g->last_slot, sizeof(t), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  out4[0] = c.n_blocks;
  out4[1] = g->d.cap_blocks;
  out4[2] = c.overflow;
  out4[3] = t.n_touched;
  return RK_OK;
}

static int finish_activation(rk_grid* g, cudaStream_t st) {
  g->last_slot = 0;
  k_assign_slots<<<1, kAssignThreads, 0, st>>>(g->d);
  RK_LAUNCHED("rk_grid activation");
  return RK_OK;
}

extern "C" int rk_grid_activate_points(rk_grid* g, const double* pts, int64_t n, double radius,
                                       void* stream) {
  cudaStream_t st = S(stream);
  k_reset_frame<<<1, 1, 0, st>>>(g->d.ctr, g->d.tc);
  if (n > 0)
    k_activate_points<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g->d, pts, n, radius,
                                                                    kEdge * g->voxel);
  return finish_activation(g, st);
}

// begin + activate + assign of one frame into touched-set slot `slot`
static int activate_image_slot(rk_grid* g, const rk_sensor* s, const float* range, const double* pose12,
                               double radius, float clip_min, float clip_max, int slot, cudaStream_t st) {
  const int n = s->dev.H * s->dev.W;
  const GridDev v = view(g, slot);
  k_begin_image_frame<<<kBeginCtas, kBeginThreads, 0, st>>>(range, n, clip_min, clip_max, v.ctr, v.tc);
  k_activate_image<<<(n + 255) / 256, 256, 0, st>>>(v, s->dev, range, pose12, radius,
                                                    kEdge * g->voxel, clip_min, clip_max);
  k_assign_slots<<<1, kAssignThreads, 0, st>>>(v);
  RK_LAUNCHED("rk_grid activation");
  return RK_OK;
}

extern "C" int rk_grid_activate_image(rk_grid* g, const rk_sensor* s, const float* range,
                                      const double* pose12, double radius, float clip_min,
                                      float clip_max, void* stream) {
  g->last_slot = 0;
  return activate_image_slot(g, s, range, pose12, radius, clip_min, clip_max, 0, S(stream));
}

extern "C" int rk_grid_set_touched(rk_grid* g, const int32_t* keys, int64_t n, void* stream) {
  cudaStream_t st = S(stream);
  g->last_slot = 0;
  k_reset_frame<<<1, 1, 0, st>>>(g->d.ctr, g->d.tc);
  if (n > 0) k_set_touched<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g->d, keys, n);
  RK_LAUNCHED("k_set_touched");
  return RK_OK;
}

static int integrate_slot(rk_grid* g, const rk_sensor* s, const float* range, const double* inv12,
                          float clip_min, float clip_max, int math, int64_t* updated, int slot,
                          cudaStream_t st, const long long* global_touch) {
  IntegrateArgs a;
  a.g = view(g, slot);
  a.s = s->dev;
  a.range = range;
  a.inv12 = inv12;
  a.voxel = g->voxel;
  a.block_ext = kEdge * g->voxel;
  a.tau = (float)g->trunc;
  a.max_w = g->max_weight;
  a.cmin = clip_min;
  a.cmax = clip_max;
  a.free_space = g->free_space;
  a.updated = reinterpret_cast<long long*>(updated);
  a.global_touch = global_touch;
  constexpr int NT = kIntegrateThreads;
  const unsigned grid = (unsigned)(num_sms() * kIntegrateCtasPerSm);
  const size_t smem = kLatticeBytes;
  const bool tab = s->dev.H <= kMaxRowsSmem && s->dev.K <= kMaxInvSmem;
  if (math == MATH_CR)
    tab ? k_integrate<MATH_CR, NT, true><<<grid, NT, smem, st>>>(a)
        : k_integrate<MATH_CR, NT, false><<<grid, NT, smem, st>>>(a);
  else if (math == MATH_NP)
    tab ? k_integrate<MATH_NP, NT, true><<<grid, NT, smem, st>>>(a)
        : k_integrate<MATH_NP, NT, false><<<grid, NT, smem, st>>>(a);
  else
    tab ? k_integrate<MATH_FAST, NT, true><<<grid, NT, smem, st>>>(a)
        : k_integrate<MATH_FAST, NT, false><<<grid, NT, smem, st>>>(a);
  RK_LAUNCHED("k_integrate");
  return RK_OK;
}

extern "C" int rk_grid_integrate(rk_grid* g, const rk_sensor* s, const float* range,
                                 const double* inv12, float clip_min, float clip_max, int math,
                                 int64_t* updated, void* stream) {
  return integrate_slot(g, s, range, inv12, clip_min, clip_max, math, updated, g->last_slot,
                        S(stream), g->global_touch);
}

// F frames: activation of frame f+1 (side stream) overlaps the integration of
// frame f (caller's stream).  Frame f uses touched-set slot f & 1; the
// activation of f+2 waits for the integration of f (same slot), the
// integration of f waits for its own activation.  Stream-capture safe (the
// side stream forks from and joins the caller's stream through events).
extern "C" int rk_grid_integrate_frames(rk_grid* g, const rk_sensor* s, const float* frames,
                                        int32_t n_frames, const double* poses12, const double* invs12,
                                        double radius, float clip_min, float clip_max, int math,
                                        int64_t* updated, void* stream) {
  cudaStream_t st = S(stream);
  if (n_frames <= 0) return RK_OK;
  const size_t px = (size_t)s->dev.H * s->dev.W;
  RK_CUDA(cudaEventRecord(g->ev_fork, st));
  RK_CUDA(cudaStreamWaitEvent(g->side, g->ev_fork, 0));
  for (int f = 0; f < n_frames; ++f) {
    const int slot = f & 1;
    if (f >= 2) RK_CUDA(cudaStreamWaitEvent(g->side, g->ev_int[slot], 0));
    int rc = activate_image_slot(g, s, frames + f * px, poses12 + 12 * f, radius, clip_min, clip_max,
                                 slot, g->side);
    if (rc) return rc;
    RK_CUDA(cudaEventRecord(g->ev_act[slot], g->side));
    RK_CUDA(cudaStreamWaitEvent(st, g->ev_act[slot], 0));
    rc = integrate_slot(g, s, frames + f * px, invs12 + 12 * f, clip_min, clip_max, math, updated,
                        slot, st, nullptr);
    if (rc) return rc;
    RK_CUDA(cudaEventRecord(g->ev_int[slot], st));
  }
  // join: the caller's stream already waited for the last activation; make
  // the side stream's tail (nothing after it) part of the caller's order too
  RK_CUDA(cudaEventRecord(g->ev_act[0], g->side));
  RK_CUDA(cudaStreamWaitEvent(st, g->ev_act[0], 0));
  g->last_slot = (n_frames - 1) & 1;
  return RK_OK;
}

// ---- batched activation for hash-sharded multi-GPU grids: all F frames are
// activated first (one touched-set slot each), their {count, max key} pairs
// reduced across ranks in ONE collective, then all F frames integrated.
extern "C" int rk_grid_reserve_slots(rk_grid* g, int32_t n, void* stream) {
  if (n <= g->n_slots) return RK_OK;
  cudaStream_t st = S(stream);
  RK_CUDA(cudaStreamSynchronize(st));
  int32_t* touched = nullptr;
  TouchCounters* tc = nullptr;
  RK_CUDA(cudaMalloc(&touched, (size_t)n * g->hash_cap * sizeof(int32_t)));
  RK_CUDA(cudaMalloc(&tc, n * sizeof(TouchCounters)));
  RK_CUDA(cudaMemset(tc, 0, n * sizeof(TouchCounters)));
  RK_CUDA(cudaMemcpy(touched, g->d.touched, (size_t)g->n_slots * g->hash_cap * sizeof(int32_t),
                     cudaMemcpyDeviceToDevice));
  RK_CUDA(cudaMemcpy(tc, g->d.tc, g->n_slots * sizeof(TouchCounters), cudaMemcpyDeviceToDevice));
  cudaFree(g->d.touched);
  cudaFree(g->d.tc);
  g->d.touched = touched;
  g->d.tc = tc;
  g->n_slots = n;
  return RK_OK;
}

extern "C" int rk_grid_activate_frames(rk_grid* g, const rk_sensor* s, const float* frames,
                                       int32_t n_frames, const double* poses12, double radius,
                                       float clip_min, float clip_max, void* stream) {
  if (n_frames > g->n_slots) {
    rk_set_error("%d frames need rk_grid_reserve_slots (have %d slots)", n_frames, g->n_slots);
    return RK_EGENERIC;
  }
  const size_t px = (size_t)s->dev.H * s->dev.W;
  for (int f = 0; f < n_frames; ++f) {
    const int rc = activate_image_slot(g, s, frames + f * px, poses12 + 12 * f, radius, clip_min,
                                       clip_max, f, S(stream));
    if (rc) return rc;
  }
  g->last_slot = n_frames > 0 ? n_frames - 1 : 0;
  return RK_OK;
}

__global__ void k_touch_stats_frames(const TouchCounters* t, int n, long long* out) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  out[2 * f] = t[f].n_touched;
  out[2 * f + 1] = (long long)t[f].max_touched_key;
}

extern "C" int rk_grid_touch_stats_frames(rk_grid* g, int32_t n_frames, int64_t* out2n, void* stream) {
  if (n_frames <= 0) return RK_OK;
  k_touch_stats_frames<<<(n_frames + 127) / 128, 128, 0, S(stream)>>>(
      g->d.tc, n_frames, reinterpret_cast<long long*>(out2n));
  RK_LAUNCHED("k_touch_stats_frames");
  return RK_OK;
}

extern "C" int rk_grid_integrate_activated(rk_grid* g, const rk_sensor* s, const float* frames,
                                           int32_t n_frames, const double* invs12,
                                           const int64_t* global2n, float clip_min, float clip_max,
                                           int math, int64_t* updated, void* stream) {
  const size_t px = (size_t)s->dev.H * s->dev.W;
  const long long* glob = reinterpret_cast<const long long*>(global2n);
  for (int f = 0; f < n_frames; ++f) {
    const int rc = integrate_slot(g, s, frames + f * px, invs12 + 12 * f, clip_min, clip_max, math,
                                  updated, f, S(stream), glob ? glob + 2 * f : nullptr);
    if (rc) return rc;
  }
  return RK_OK;
}

extern "C" int rk_grid_keys(rk_grid* g, int touched_only, int32_t* keys_out, int64_t cap,
                            int64_t* n_host, void* stream) {
  cudaStream_t st = S(stream);
  Counters c;
  TouchCounters t;
  RK_CUDA(cudaMemcpyAsync(&c, g->d.ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaMemcpyAsync(&t, g->d.tc + g->last_slot, sizeof(t), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  long long n = touched_only ? t.n_touched : c.n_blocks;
  if (n_host) *n_host = n;
  if (keys_out && cap > 0 && n > 0) {
    if (touched_only) k_keys_touched<<<128, 256, 0, st>>>(view(g, g->last_slot), keys_out, cap);
    else k_keys_all<<<128, 256, 0, st>>>(g->d, keys_out, cap);
    RK_LAUNCHED("rk_grid_keys");
  }
  return RK_OK;
}

extern "C" int rk_grid_read_blocks(rk_grid* g, const int32_t* keys, int64_t n, float* vox,
                                   uint8_t* found, void* stream) {
  if (n <= 0) return RK_OK;
  k_read_blocks<<<(unsigned)n, 256, 0, S(stream)>>>(g->d, keys, n, reinterpret_cast<float2*>(vox), found);
  RK_LAUNCHED("k_read_blocks");
  return RK_OK;
}

extern "C" int rk_grid_write_blocks(rk_grid* g, const int32_t* keys, int64_t n, const float* vox,
                                    void* stream) {
  cudaStream_t st = S(stream);
  if (n <= 0) return RK_OK;
  k_reset_frame<<<1, 1, 0, st>>>(g->d.ctr, g->d.tc);
  k_insert_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g->d, keys, n);
  int rc = finish_activation(g, st);
  if (rc) return rc;
  k_write_blocks<<<(unsigned)n, 256, 0, st>>>(g->d, keys, n, reinterpret_cast<const float2*>(vox));
  RK_LAUNCHED("k_write_blocks");
  return RK_OK;
}

extern "C" int rk_grid_query(rk_grid* g, const double* pts, int64_t n, double* sdf, double* weight,
                             uint8_t* observed, void* stream) {
  if (n <= 0) return RK_OK;
  k_query<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(g->d, g->voxel, pts, n, sdf, weight,
                                                               observed);
  RK_LAUNCHED("k_query");
  return RK_OK;
}

int rk_grid_view_(rk_grid* g, GridView* v) {
  Counters c;
  RK_CUDA(cudaMemcpy(&c, g->d.ctr, sizeof(c), cudaMemcpyDeviceToHost));
  v->vox = g->d.vox;
  v->block_keys = g->d.block_keys;
  v->h_keys = g->d.h_keys;
  v->h_slot = g->d.h_slot;
  v->hash_mask = g->d.hash_mask;
  v->n_blocks = c.n_blocks;
  v->shard_rank = g->d.shard_rank;
  v->shard_world = g->d.shard_world;
  return RK_OK;
}

double rk_grid_voxel_(rk_grid* g) { return g->voxel; }

namespace {
__global__ void k_clear_blocks(GridDev g) {
  const long long nb = g.ctr->n_blocks;
  float4* v = reinterpret_cast<float4*>(g.vox);
  const long long n4 = nb * (kVox / 2);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__global__ void k_clear_counters(Counters* c, TouchCounters* t, int n_slots) {
  c->n_blocks = 0;
  c->n_fresh = 0;
  c->overflow = 0;
  c->updated = 0;
  c->n_points = 0;
  for (int i = 0; i < n_slots; ++i) {
    t[i].n_touched = 0;
    t[i].max_touched_key = 0ull;
  }
}
}  // namespace

// empty the grid without freeing it (async; keeps capacity)
extern "C" int rk_grid_clear(rk_grid* g, void* stream) {
  cudaStream_t st = S(stream);
  k_clear_blocks<<<148 * 8, 256, 0, st>>>(g->d);
  RK_CUDA(cudaMemsetAsync(g->d.h_keys, 0xff, g->hash_cap * sizeof(unsigned long long), st));
  RK_CUDA(cudaMemsetAsync(g->d.h_slot, 0xff, g->hash_cap * sizeof(int32_t), st));
  k_clear_counters<<<1, 1, 0, st>>>(g->d.ctr, g->d.tc, g->n_slots);
  RK_LAUNCHED("rk_grid_clear");
  return RK_OK;
}

// multi-GPU hash sharding: from now on this grid only allocates blocks with
// rk_owner_mix(packed key) % world == rank
extern "C" int rk_grid_set_shard(rk_grid* g, int32_t rank, int32_t world) {
  if (world < 1 || rank < 0 || rank >= world) {
    rk_set_error("bad shard rank %d / world %d", rank, world);
    return RK_EGENERIC;
  }
  g->d.shard_rank = rank;
  g->d.shard_world = world;
  return RK_OK;
}

// host mirror of the device owner function (for tests / host-side routing)
extern "C" int rk_block_owner(const int32_t* keys_host, int64_t n, int32_t world, int32_t* owner_host) {
  for (int64_t i = 0; i < n; ++i) {
    unsigned long long key = pack_key(keys_host[3 * i], keys_host[3 * i + 1], keys_host[3 * i + 2]);
    owner_host[i] = (int32_t)(rk_owner_mix(key) % (unsigned long long)world);
  }
  return RK_OK;
}

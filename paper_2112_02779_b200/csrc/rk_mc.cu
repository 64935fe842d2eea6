// rk_mc.cu -- K6: Marching Cubes over every stored block (mesh_extract.py:85-209).
//
// One CTA per block; the 27-neighbour slot table lives in shared memory so
// corner values and central-difference gradients read the neighbouring blocks
// directly (the reference's 19^3 halo, mesh_extract.py:58-82, without the
// copy).  Vertices are deduplicated globally through a hash keyed by the
// canonical (lower lattice corner, axis) of each crossed edge -- or by the
// lattice point itself when the crossing snaps onto a corner, which is exactly
// the reference's exact-position merge (mesh_extract.py:129-155).  Vertex
// positions/normals are computed from the canonical corner with the
// reference's float64 op order, so every cell that meets a vertex agrees on it
// bit for bit.  Output order differs from the reference's sequential loop
// (the parity contract is "same vertex set and triangle set up to relabelling").
#include "rk_common.cuh"

using namespace rk;

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

namespace {

constexpr int kEdge = 16;
constexpr int kVox = kEdge * kEdge * kEdge;
constexpr long long kBias = 1ll << 17;
constexpr long long kShift = 1ll << 18;
constexpr unsigned long long kEmpty = ~0ull;

// corner offsets (mc_tables.py:28-31) and canonical edges (mesh_extract.py:25-34)
__constant__ int c_corner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                   {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
__constant__ int c_canon[12][2] = {{0, 1}, {1, 2}, {3, 2}, {0, 3}, {4, 5}, {5, 6},
                                   {7, 6}, {4, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
__constant__ int c_axis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__device__ int slot_of(const GridView& g, long long x, long long y, long long z) {
  unsigned long long key = (unsigned long long)(((x + kBias) * kShift + (y + kBias)) * kShift + (z + kBias));
  unsigned long long h = mix64(key) & g.hash_mask;
  for (int probe = 0; probe < 4096; ++probe) {
    unsigned long long k = g.h_keys[h];
    if (k == key) return g.h_slot[h];
    if (k == kEmpty) return -1;
    h = (h + 1) & g.hash_mask;
  }
  return -1;
}

struct Mesh {
  unsigned long long* vkeys;  // vertex hash keys
  int32_t* vids;              // vertex hash values
  unsigned long long vmask;
  double* verts;  // (vcap, 3)
  double* nrms;   // (vcap, 3)
  int32_t* tris;  // (tcap, 3)
  long long vcap, tcap;
  unsigned long long* counters;  // [0] vertices, [1] triangles, [2] active cells, [3] tri upper, [4] overflow
};

// corner sample (d, w) at block-local lattice coords in [-1, 17]
__device__ __forceinline__ float2 sample(const GridView& g, const int* nb, int x, int y, int z) {
  int ox = x < 0 ? 0 : (x >= kEdge ? 2 : 1);
  int oy = y < 0 ? 0 : (y >= kEdge ? 2 : 1);
  int oz = z < 0 ? 0 : (z >= kEdge ? 2 : 1);
  int slot = nb[(ox * 3 + oy) * 3 + oz];
  if (slot < 0) return make_float2(0.f, 0.f);
  int lx = x - (ox - 1) * kEdge, ly = y - (oy - 1) * kEdge, lz = z - (oz - 1) * kEdge;
  RK_DCHECK(lx >= 0 && lx < kEdge && ly >= 0 && ly < kEdge && lz >= 0 && lz < kEdge && slot < g.n_blocks,
            "K6 corner sample", slot, (lx * kEdge + ly) * kEdge + lz);
  return g.vox[(size_t)slot * kVox + (lx * kEdge + ly) * kEdge + lz];
}

// a hash-sharded grid (rk_grid_set_shard) meshes only the blocks it owns;
// blocks it holds as halo copies of other ranks' blocks only feed the samples
__device__ __forceinline__ bool foreign_block(const GridView& g, int slot) {
  if (g.shard_world <= 1) return false;
  const int4 k = g.block_keys[slot];
  return rk_block_owner_of(k.x, k.y, k.z, g.shard_world) != g.shard_rank;
}

__device__ __forceinline__ void load_neighbours(const GridView& g, int slot, int* nb) {
  if (threadIdx.x < 27) {
    int4 k = g.block_keys[slot];
    int t = threadIdx.x;
    nb[t] = slot_of(g, k.x + t / 9 - 1, k.y + (t / 3) % 3 - 1, k.z + t % 3 - 1);
  }
  __syncthreads();
}

// case index of a cell, or -1 when the cell is not active
__device__ __forceinline__ int cell_case(const GridView& g, const int* nb, int lx, int ly, int lz,
                                         float min_w, double vals[8]) {
  int cs = 0;
  bool full = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    float2 s = sample(g, nb, lx + c_corner[c][0], ly + c_corner[c][1], lz + c_corner[c][2]);
    vals[c] = (double)s.x;
    full = full && s.y >= min_w;
    cs |= (s.x < 0.0f ? 1 : 0) << c;
  }
  return (full && cs > 0 && cs < 255) ? cs : -1;
}

__global__ void k_mc_count(GridView g, const int8_t* __restrict__ table, float min_w,
                           unsigned long long* counters) {
  if (foreign_block(g, blockIdx.x)) return;  // uniform per CTA
  __shared__ int nb[27];
  __shared__ int8_t tab[256 * 16];
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) tab[i] = table[i];
  load_neighbours(g, blockIdx.x, nb);
  unsigned long long act = 0, tri = 0;
  for (int cell = threadIdx.x; cell < kVox; cell += blockDim.x) {
    double vals[8];
    int cs = cell_case(g, nb, cell >> 8, (cell >> 4) & 15, cell & 15, min_w, vals);
    if (cs < 0) continue;
    ++act;
    for (int i = 0; i < 16 && tab[cs * 16 + i] >= 0; i += 3) ++tri;
  }
  act = __reduce_add_sync(0xffffffffu, (unsigned)act);
  tri = __reduce_add_sync(0xffffffffu, (unsigned)tri);
  if ((threadIdx.x & 31) == 0) {
    if (act) atomicAdd(counters + 2, act);
    if (tri) atomicAdd(counters + 3, tri);
  }
}

__device__ __forceinline__ unsigned long long vkey(long long x, long long y, long long z, int kind) {
  const long long b = 1ll << 19;
  return ((unsigned long long)(x + b) << 42) | ((unsigned long long)(y + b) << 22) |
         ((unsigned long long)(z + b) << 2) | (unsigned long long)kind;
}

// central / one-sided / zero difference at block-local lattice point p (181-199)
__device__ __forceinline__ double grad_axis(const GridView& g, const int* nb, int px, int py, int pz,
                                            int ax, double voxel) {
  int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  float2 c = sample(g, nb, px, py, pz);
  float2 hi = sample(g, nb, px + dx, py + dy, pz + dz);
  float2 lo = sample(g, nb, px - dx, py - dy, pz - dz);
  bool hok = hi.y > 0.f, lok = lo.y > 0.f;
  double d = c.x, h = hi.x, l = lo.x;
  if (hok && lok) return __ddiv_rn(__dsub_rn(h, l), 2.0 * voxel);
  if (hok) return __ddiv_rn(__dsub_rn(h, d), voxel);
  if (lok) return __ddiv_rn(__dsub_rn(d, l), voxel);
  return 0.0;
}

// insert the vertex of edge e of a cell; returns its id
__device__ int vertex_of(const GridView& g, const Mesh& m, const int* nb, int4 bk, int lx, int ly,
                         int lz, int e, const double vals[8], double voxel) {
  const int a = c_canon[e][0], b = c_canon[e][1];
  const double da = vals[a], db = vals[b];
  double t = fabs(__dsub_rn(da, db)) < 1e-9 ? 0.5 : __ddiv_rn(da, __dsub_rn(da, db));
  if (t < 1e-6) t = 0.0;
  else if (t > 1.0 - 1e-6) t = 1.0;
  const int ax = lx + c_corner[a][0], ay = ly + c_corner[a][1], az = lz + c_corner[a][2];
  const int bx = lx + c_corner[b][0], by = ly + c_corner[b][1], bz = lz + c_corner[b][2];
  const long long gx = (long long)bk.x * kEdge, gy = (long long)bk.y * kEdge, gz = (long long)bk.z * kEdge;
  unsigned long long key;
  if (t == 0.0) key = vkey(gx + ax, gy + ay, gz + az, 3);
  else if (t == 1.0) key = vkey(gx + bx, gy + by, gz + bz, 3);
  else key = vkey(gx + ax, gy + ay, gz + az, c_axis[e]);
  unsigned long long h = mix64(key) & m.vmask;
  for (long long probe = 0; probe <= (long long)m.vmask; ++probe) {
    unsigned long long k = *((volatile unsigned long long*)(m.vkeys + h));
    if (k == key) break;
    if (k == kEmpty) {
      unsigned long long prev = atomicCAS(m.vkeys + h, kEmpty, key);
      if (prev == kEmpty) {
        // first owner: allocate the id and write the vertex
        unsigned long long id = atomicAdd(m.counters + 0, 1ull);
        if ((long long)id >= m.vcap) {
          atomicExch(m.counters + 4, 1ull);
          atomicExch(m.vids + h, -2);  // release waiters
          return -2;
        }
        double pos[3], nrm[3];
        const double pa[3] = {(double)(gx + ax), (double)(gy + ay), (double)(gz + az)};
        const double pb[3] = {(double)(gx + bx), (double)(gy + by), (double)(gz + bz)};
        for (int c = 0; c < 3; ++c) {
          double qa = __dmul_rn(__dadd_rn(pa[c], 0.5), voxel);
          double qb = __dmul_rn(__dadd_rn(pb[c], 0.5), voxel);
          pos[c] = __dadd_rn(__dmul_rn(qa, __dsub_rn(1.0, t)), __dmul_rn(qb, t));
          double ga = grad_axis(g, nb, ax, ay, az, c, voxel);
          double gb = grad_axis(g, nb, bx, by, bz, c, voxel);
          nrm[c] = __dadd_rn(__dmul_rn(ga, __dsub_rn(1.0, t)), __dmul_rn(gb, t));
        }
        for (int c = 0; c < 3; ++c) {
          m.verts[3 * id + c] = pos[c];
          m.nrms[3 * id + c] = nrm[c];
        }
        __threadfence();
        atomicExch(m.vids + h, (int)id);
        return (int)id;
      }
      if (prev == key) break;
    }
    h = (h + 1) & m.vmask;
  }
  // another thread owns the key: wait for it to publish the id
  int id;
#if RK_DEBUG_CHECKS
  long long spins = 0;
#endif
  while ((id = *((volatile int*)(m.vids + h))) == -1) {
#if RK_DEBUG_CHECKS
    RK_DCHECK(++spins < (1ll << 28), "K6 vertex publish wait", (long long)h, spins);
#endif
  }
  RK_DCHECK(id == -2 || (id >= 0 && id < m.vcap), "K6 vertex id", id, m.vcap);
  return id;
}

__global__ void k_mc_vertices(GridView g, const int8_t* __restrict__ table, float min_w, double voxel,
                              Mesh m) {
  if (foreign_block(g, blockIdx.x)) return;
  __shared__ int nb[27];
  __shared__ int8_t tab[256 * 16];
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) tab[i] = table[i];
  load_neighbours(g, blockIdx.x, nb);
  const int4 bk = g.block_keys[blockIdx.x];
  for (int cell = threadIdx.x; cell < kVox; cell += blockDim.x) {
    const int lx = cell >> 8, ly = (cell >> 4) & 15, lz = cell & 15;
    double vals[8];
    int cs = cell_case(g, nb, lx, ly, lz, min_w, vals);
    if (cs < 0) continue;
    unsigned done = 0;
    for (int i = 0; i < 16; ++i) {
      int e = tab[cs * 16 + i];
      if (e < 0) break;
      if (done & (1u << e)) continue;
      done |= 1u << e;
      vertex_of(g, m, nb, bk, lx, ly, lz, e, vals, voxel);
    }
  }
}

__device__ __forceinline__ int find_vertex(const Mesh& m, unsigned long long key) {
  unsigned long long h = mix64(key) & m.vmask;
  for (long long probe = 0; probe <= (long long)m.vmask; ++probe) {
    unsigned long long k = m.vkeys[h];
    if (k == key) return m.vids[h];
    if (k == kEmpty) return -1;
    h = (h + 1) & m.vmask;
  }
  return -1;
}

__global__ void k_mc_triangles(GridView g, const int8_t* __restrict__ table, float min_w, Mesh m) {
  if (foreign_block(g, blockIdx.x)) return;
  __shared__ int nb[27];
  __shared__ int8_t tab[256 * 16];
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) tab[i] = table[i];
  load_neighbours(g, blockIdx.x, nb);
  const int4 bk = g.block_keys[blockIdx.x];
  const long long gx = (long long)bk.x * kEdge, gy = (long long)bk.y * kEdge, gz = (long long)bk.z * kEdge;
  for (int cell = threadIdx.x; cell < kVox; cell += blockDim.x) {
    const int lx = cell >> 8, ly = (cell >> 4) & 15, lz = cell & 15;
    double vals[8];
    int cs = cell_case(g, nb, lx, ly, lz, min_w, vals);
    if (cs < 0) continue;
    for (int i = 0; i < 16; i += 3) {
      if (tab[cs * 16 + i] < 0) break;
      int id[3];
      for (int j = 0; j < 3; ++j) {
        int e = tab[cs * 16 + i + j];
        const int a = c_canon[e][0], b = c_canon[e][1];
        const double da = vals[a], db = vals[b];
        double t = fabs(__dsub_rn(da, db)) < 1e-9 ? 0.5 : __ddiv_rn(da, __dsub_rn(da, db));
        unsigned long long key;
        if (t < 1e-6)
          key = vkey(gx + lx + c_corner[a][0], gy + ly + c_corner[a][1], gz + lz + c_corner[a][2], 3);
        else if (t > 1.0 - 1e-6)
          key = vkey(gx + lx + c_corner[b][0], gy + ly + c_corner[b][1], gz + lz + c_corner[b][2], 3);
        else
          key = vkey(gx + lx + c_corner[a][0], gy + ly + c_corner[a][1], gz + lz + c_corner[a][2], c_axis[e]);
        id[j] = find_vertex(m, key);
      }
      if (id[0] < 0 || id[1] < 0 || id[2] < 0) continue;
      if (id[0] == id[1] || id[1] == id[2] || id[0] == id[2]) continue;
      RK_DCHECK(id[0] < m.vcap && id[1] < m.vcap && id[2] < m.vcap, "K6 triangle vertex", id[0], m.vcap);
      // area test on the final positions (mesh_extract.py:202-209)
      const double* A = m.verts + 3 * id[0];
      const double* B = m.verts + 3 * id[1];
      const double* Cc = m.verts + 3 * id[2];
      double u0 = __dsub_rn(B[0], A[0]), u1 = __dsub_rn(B[1], A[1]), u2 = __dsub_rn(B[2], A[2]);
      double v0 = __dsub_rn(Cc[0], A[0]), v1 = __dsub_rn(Cc[1], A[1]), v2 = __dsub_rn(Cc[2], A[2]);
      double c0 = __dsub_rn(__dmul_rn(u1, v2), __dmul_rn(u2, v1));
      double c1 = __dsub_rn(__dmul_rn(u2, v0), __dmul_rn(u0, v2));
      double c2 = __dsub_rn(__dmul_rn(u0, v1), __dmul_rn(u1, v0));
      double area2 = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(c0, c0), __dmul_rn(c1, c1)), __dmul_rn(c2, c2)));
      if (!(area2 > 2e-12)) continue;
      unsigned long long slot = atomicAdd(m.counters + 1, 1ull);
      if ((long long)slot >= m.tcap) { atomicExch(m.counters + 4, 1ull); continue; }
      m.tris[3 * slot] = id[0];
      m.tris[3 * slot + 1] = id[1];
      m.tris[3 * slot + 2] = id[2];
    }
  }
}

__global__ void k_mc_normalize(Mesh m, long long nv) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nv) return;
  double* n = m.nrms + 3 * i;
  double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(n[0], n[0]), __dmul_rn(n[1], n[1])), __dmul_rn(n[2], n[2])));
  if (nn > 1e-12) {
    n[0] = __ddiv_rn(n[0], nn);
    n[1] = __ddiv_rn(n[1], nn);
    n[2] = __ddiv_rn(n[2], nn);
  } else {
    n[0] = 0.0;
    n[1] = 0.0;
    n[2] = 1.0;
  }
}

}  // namespace

// --------------------------------------------------------------- host side
// The mesh lives in a grow-only scratch owned by the grid (rk_grid_scratch_):
// valid until the next rk_mc_extract on the same grid or its destruction; no
// cudaMalloc / cudaFree (device-wide synchronisations) per extraction.
struct rk_mesh {
  Mesh m;
  long long nv, nt;
};


extern "C" int rk_mc_extract(rk_grid* grid, const int8_t* tri_table, float min_weight,
                             rk_mesh** out, void* stream) {
  cudaStream_t st = S(stream);
  GridView g;
  int rc = rk_grid_view_(grid, &g);
  if (rc) return rc;
  unsigned long long* ctr =
      static_cast<unsigned long long*>(rk_grid_scratch_(grid, 1, 8 * sizeof(unsigned long long)));
  if (!ctr) return RK_ECUDA;
  RK_CUDA(cudaMemsetAsync(ctr, 0, 8 * sizeof(unsigned long long), st));
  rk_mesh* mesh = new rk_mesh();
  mesh->nv = mesh->nt = 0;
  unsigned long long h_ctr[8] = {0};
  if (g.n_blocks > 0) {
    k_mc_count<<<(unsigned)g.n_blocks, 256, 0, st>>>(g, tri_table, min_weight, ctr);
    RK_LAUNCHED("k_mc_count");
    RK_CUDA(cudaMemcpyAsync(h_ctr, ctr, sizeof(h_ctr), cudaMemcpyDeviceToHost, st));
    RK_CUDA(cudaStreamSynchronize(st));
  }
  const long long active = (long long)h_ctr[2], tri_upper = (long long)h_ctr[3];
  // each active cell creates at most its 12 edges' vertices; edges are shared
  const long long vcap = active * 12 + 16, tcap = tri_upper + 16;
  unsigned long long hcap = 1024;
  while (hcap < (unsigned long long)vcap * 2ull) hcap <<= 1;
  size_t bytes = hcap * (sizeof(unsigned long long) + sizeof(int32_t)) + vcap * 6 * sizeof(double) +
                 tcap * 3 * sizeof(int32_t) + 1024;
  char* blob = static_cast<char*>(rk_grid_scratch_(grid, 0, bytes));
  if (!blob) {
    delete mesh;
    return RK_ECUDA;
  }
  Mesh& m = mesh->m;
  m.vkeys = reinterpret_cast<unsigned long long*>(blob);
  m.vids = reinterpret_cast<int32_t*>(m.vkeys + hcap);
  m.verts = reinterpret_cast<double*>(((uintptr_t)(m.vids + hcap) + 255) & ~uintptr_t(255));
  m.nrms = m.verts + vcap * 3;
  m.tris = reinterpret_cast<int32_t*>(m.nrms + vcap * 3);
  m.vmask = hcap - 1;
  m.vcap = vcap;
  m.tcap = tcap;
  m.counters = ctr;
  RK_CUDA(cudaMemsetAsync(m.vkeys, 0xff, hcap * sizeof(unsigned long long), st));
  RK_CUDA(cudaMemsetAsync(m.vids, 0xff, hcap * sizeof(int32_t), st));
  const double vs = rk_grid_voxel_(grid);
  if (active > 0) {
    k_mc_vertices<<<(unsigned)g.n_blocks, 256, 0, st>>>(g, tri_table, min_weight, vs, m);
    k_mc_triangles<<<(unsigned)g.n_blocks, 256, 0, st>>>(g, tri_table, min_weight, m);
    RK_LAUNCHED("k_mc_vertices/triangles");
  }
  RK_CUDA(cudaMemcpyAsync(h_ctr, ctr, sizeof(h_ctr), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  if (h_ctr[4]) {
    rk_set_error("marching cubes output overflow");
    delete mesh;
    return RK_ECAPACITY;
  }
  mesh->nv = (long long)h_ctr[0];
  mesh->nt = (long long)h_ctr[1];
  if (mesh->nv > 0) {
    k_mc_normalize<<<(unsigned)((mesh->nv + 255) / 256), 256, 0, st>>>(m, mesh->nv);
    RK_LAUNCHED("k_mc_normalize");
  }
  *out = mesh;
  return RK_OK;
}

extern "C" int rk_mesh_info(rk_mesh* mesh, int64_t* counts_host) {
  counts_host[0] = mesh->nv;
  counts_host[1] = mesh->nt;
  return RK_OK;
}

extern "C" int rk_mesh_copy(rk_mesh* mesh, double* verts, double* normals, int32_t* tris, void* stream) {
  cudaStream_t st = S(stream);
  if (mesh->nv) {
    RK_CUDA(cudaMemcpyAsync(verts, mesh->m.verts, mesh->nv * 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    RK_CUDA(cudaMemcpyAsync(normals, mesh->m.nrms, mesh->nv * 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  if (mesh->nt)
    RK_CUDA(cudaMemcpyAsync(tris, mesh->m.tris, mesh->nt * 3 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  return RK_OK;
}

extern "C" int rk_mesh_free(rk_mesh* mesh) {
  delete mesh;  // the buffers belong to the grid's scratch
  return RK_OK;
}

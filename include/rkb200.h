/*
 * rkb200.h -- C ABI of librkb200.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of rangekit (arXiv 2112.02779's range-image LiDAR
 * pipeline).  Plain pointers and sizes only: every array argument is a DEVICE
 * pointer unless its name ends in `_host`; `stream` is a cudaStream_t.
 *
 * Each entry point replaces one reference interface (file:line into
 * /root/reference/pkg/src/rangekit/).  The reference is pure Python, so the
 * "FFI" a maintainer would add is the ctypes layer shown in INTEGRATION.md;
 * the package `paper_2112_02779_b200` is exactly that layer.
 *
 * Status codes: 0 = OK, negative = error; each maps 1:1 onto a rangekit
 * exception class (errors.py:4-45, see paper_2112_02779_b200/errors.py).
 * rk_last_error() returns the message of the last failure on this thread.
 */
#ifndef RKB200_H
#define RKB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RK_OK = 0,
  RK_EGENERIC = -1,         /* RangekitError */
  RK_EINTRINSICS = -2,      /* InvalidIntrinsics */
  RK_EOUTOFFOV = -3,        /* OutOfFov */
  RK_EDEGENERATE_RANGE = -4,/* DegenerateRange */
  RK_EEMPTY = -5,           /* EmptyInput */
  RK_EMISSING_NORMALS = -6, /* MissingNormals */
  RK_EDEGENERATE_GEOM = -7, /* DegenerateGeometry */
  RK_EINVALID_POSE = -8,    /* InvalidPose */
  RK_EFORMAT = -9,          /* FormatError */
  RK_ECUDA = -10,           /* CUDA launch / allocation failure */
  RK_ECAPACITY = -11        /* voxel-block pool full (caller grows, retries) */
};

/* math modes of the float32 projection:
 * FAST = minimax atan2/asin + reciprocal refinements (and a float32 ICP move),
 * CR = float64 transcendentals rounded once (bit-comparable with the oracle's
 * math="cr"), LIBM = CUDA's accurate atan2f/asinf with IEEE division (only
 * rk_project_f32 accepts it), NP = numpy's own float32 arctan2/arcsin (the
 * SVML sequences restated bit for bit) with exact arithmetic everywhere else:
 * the reference's projection (lidar_model.py:262-344) bit for bit. */
enum { RK_MATH_FAST = 0, RK_MATH_CR = 1, RK_MATH_LIBM = 2, RK_MATH_NP = 3 };
/* rk_project_f32 only (test hook): RK_MATH_NP through the finite-operand
 * variant K3 and K5 use (branch-free square root, NaN-free clamps) -- equal
 * to RK_MATH_NP bit for bit on finite points */
#define RK_MATH_NP_FINITE 4

/* per-pair ICP status (registration.py:266-272) */
enum { RK_ICP_CONVERGED = 0, RK_ICP_TOO_FEW = 1, RK_ICP_DEGENERATE = 2, RK_ICP_BAD_PAIR = 3 };

typedef struct rk_sensor rk_sensor; /* device-resident sensor tables   */
typedef struct rk_grid rk_grid;     /* device voxel-block hash + pool  */

/* ------------------------------------------------------------ misc */
int rk_last_error(char* buf_host, size_t cap);
int rk_version(void);
/* sizeof the ABI structs (0: rk_sensor_desc, 1: rk_icp_config; -1 otherwise):
 * a binding checks its struct mirrors against these at load time */
int rk_struct_size(int which);

/* ------------------------------------------------------------ sensor
 * Replaces LidarIntrinsics' cached tables (lidar_model.py:94-179): the host
 * builds them with the reference's numpy expressions and uploads them once. */
typedef struct {
  int32_t height, width;
  double receiver_radius;
  const double* dirs_host;      /* (H*W*3) float64 ray_dirs               */
  const double* origins_host;   /* (W*3)  float64 ray_origins            */
  const double* azimuth_host;   /* (H)                                    */
  const double* elevation_host; /* (H)                                    */
  const int32_t* inv_rows_host; /* (inv_size) InverseElevationLut.rows    */
  int32_t inv_size;
  double inv_phi_min, inv_phi_max;
  double fov_lo, fov_hi;        /* LidarIntrinsics.fov_bounds             */
} rk_sensor_desc;

int rk_sensor_create(const rk_sensor_desc* desc, rk_sensor** out);
int rk_sensor_destroy(rk_sensor* s);

/* project_many(single=True, refine=False)  lidar_model.py:262-344 */
int rk_project_f32(const rk_sensor* s, const float* pts, int64_t n, int math,
                   float* u, int32_t* v, float* r, int8_t* status, void* stream);
/* diagnostic: RK_MATH_NP's arithmetic elementwise on device arrays --
 * fn 0: out = np.arctan2(a, b) (lidar_model.py:288), fn 1: out = np.arcsin(a)
 * (lidar_model.py:45; |a| <= 1), fn 2: the kernels' range-check-free
 * division a / b, fn 3: IEEE a / b, fn 4: the kernels' square root for
 * operands in [2^-101, 2^128), fn 5: IEEE sqrt(a); float32 (parity tests) */
int rk_svml_eval(const rk_sensor* s, int fn, const float* a, const float* b, int64_t n,
                 float* out, void* stream);
/* project_many(single=False) float64 fixed-point path, lidar_model.py:287-344.
 * work: caller scratch of >= 3*n doubles + 16 bytes. */
int rk_project_f64(const rk_sensor* s, const double* pts, int64_t n, int max_iters,
                   double tol, int refine, double* u, int32_t* v, double* r,
                   int8_t* status, double* work, void* stream);
/* LidarIntrinsics.row_from_elevation  lidar_model.py:181-202 (is_f64 selects dtype) */
int rk_row_from_elevation(const rk_sensor* s, const void* phi, int is_f64, int64_t n,
                          int32_t* v, void* stream);
/* InverseElevationLut.lookup  lidar_model.py:60-66 (stand-alone table) */
int rk_inverse_lut_lookup(const int32_t* rows, int32_t k, double phi_min, double phi_max,
                          const void* phi, int is_f64, int64_t n, int32_t* out, void* stream);
/* unproject_many  lidar_model.py:236-250 */
int rk_unproject_many(const rk_sensor* s, const double* u, const int64_t* v,
                      const double* r, int64_t n, double* out, void* stream);

/* ------------------------------------------------------------ range images
 * unproject_image  range_image.py:129-133 : (B,H,W) float32 -> (B,H,W,3) float64 */
int rk_unproject_image(const rk_sensor* s, const float* range, int32_t batch,
                       double* out, void* stream);
/* compute_normal_map(method="cross")  range_image.py:197-240.  Any output may
 * be NULL.  surfel = {nx, ny, nz, range if valid else 0} (the ICP gather map). */
int rk_normals_cross(const rk_sensor* s, const float* range, int32_t batch,
                     float* normals, uint8_t* valid, float* surfel, void* stream);
/* compute_normal_map(method="pca")  range_image.py:243-283: smallest
 * covariance eigenvector over the (2*radius+1)^2 window's valid neighbours
 * within disc_abs + disc_rel * r; outputs as rk_normals_cross (any may be NULL). */
int rk_normals_pca(const rk_sensor* s, const float* range, int32_t batch, int32_t radius,
                   double disc_abs, double disc_rel, float* normals, uint8_t* valid, float* surfel,
                   void* stream);
/* from_point_cloud's z-buffer  range_image.py:170-194: given rk_project_f64's
 * (u, v, r, status) of n points, the (H,W) float32 image of the nearest range
 * per pixel (0 = empty) and stats4 = {kept, collisions, out_of_fov, degenerate}
 * (device int64[4]).  zwork: H*W 64-bit scratch. */
int rk_zbuffer_image(const rk_sensor* s, const double* u, const int32_t* v, const double* r,
                     const int8_t* status, int64_t n, float* range_out, int64_t* stats4,
                     unsigned long long* zwork, void* stream);
/* rk_normals_cross's surfel map as a pyramid of per-pixel records, per
 * image: the full map (H*W records) followed by the decimated map of every
 * stride in strides_host that is > 1 (ceil(H/s) x ceil(W/s), pixel (i, j) =
 * full (i*s, j*s)), in order; pitch (in records) = H*W + sum of the decimated
 * sizes.  The registration's coarse levels gather from compact maps.  A
 * record is rk_surfel_record_floats() floats: 4 = {nx, ny, nz,
 * range-if-valid} (default build; the association target is formed from the
 * sensor's shared float32 ray tables), 8 = that plus {target r*dir32 +
 * origin32, 0} (RK_SURFEL_REC=32 builds). */
int rk_surfel_record_floats(void);
int rk_normals_cross_pyramid(const rk_sensor* s, const float* range, int32_t batch,
                             const int32_t* strides_host, int32_t n_strides, float* surfel_pyr,
                             int64_t pitch, void* stream);
/* StridedView + points_at_stride / to_point_cloud mask, range_image.py:69-157:
 * row-major flat base-pixel indices (v*W+u) of the stride-s view whose range
 * passes r>0 & clip_min<=r<=clip_max, per image; idx has capacity
 * ceil(H/s)*ceil(W/s) per image, count[b] receives the length. */
int rk_stride_compact(const rk_sensor* s, const float* range, int32_t batch, int32_t stride,
                      float clip_min, float clip_max, int32_t* idx, int32_t* count,
                      void* stream);
/* _unproject_pixels  range_image.py:160-167 : gather idx[0..n) of one image */
int rk_unproject_pixels(const rk_sensor* s, const float* range, const int32_t* idx,
                        const int32_t* count, int64_t cap, double* out, void* stream);
/* stable compaction of a uint8 mask: idx[0..count) = flatnonzero(mask) */
int rk_compact_mask(const uint8_t* mask, int64_t n, int32_t* idx, int32_t* count,
                    void* stream);

/* ------------------------------------------------------------ registration */
typedef struct {
  double kernel_scale;     /* RegistrationConfig.kernel_scale            */
  double max_dist;         /* RegistrationConfig.max_correspondence_dist */
  double rot_eps, trans_eps;
  float clip_min, clip_max;
  int32_t n_levels;
  int32_t strides[8];
  int32_t iters[8];
  int32_t min_corr;
  int32_t scale_with_stride;
  int32_t math;            /* RK_MATH_* */
  /* destination surfel layout: 0 = one (H*W) map per image, gathered at
   * stride-aligned pixels; else the per-image pitch (pixels) of a surfel
   * pyramid (rk_normals_cross_pyramid) and, per level, the pixel offset of
   * its decimated map (< 0: use the full-resolution map at offset 0). */
  int64_t surfel_pitch;
  int32_t surfel_level_off[8];
  /* image-pool sizes: a pair whose pair_src / pair_dst index lies outside
   * [0, n) is not registered and gets status RK_ICP_BAD_PAIR (out12 = its
   * init pose); 0 = unchecked */
  int32_t n_src_images, n_dst_images;
} rk_icp_config;

/* projective_correspondences(single=True)  registration.py:117-187 for one
 * (source cloud, destination image) pair: keep[i] = 1 for surviving points,
 * target/normal (n*3 float32) filled where keep. pose = [R row-major, t]. */
int rk_correspondences_f32(const rk_sensor* s, const double* src_pts, int64_t n,
                           const float* dst_range, const float* dst_surfel,
                           const double* pose12, double max_dist, int32_t stride,
                           int math, uint8_t* keep, float* target, float* normal,
                           void* stream);

/* surfel map {n, range-if-valid} from an explicit NormalImage (vectors, valid) */
int rk_make_surfel(const float* range, const float* normals, const uint8_t* valid, int64_t n,
                   float* surfel, void* stream);

/* register() over a batch of independent pairs  registration.py:237-289.
 * src_range/dst_range: pools of (H,W) float32 images; pair b registers
 * src_range[pair_src[b]] to dst_range[pair_dst[b]] using dst_surfel[pair_dst[b]]
 * (rk_normals_cross output).  init12/out12: (B,12) float64.  status: RK_ICP_*.
 * stats (may be NULL): (B, max_total_iters, 5) float64 rows
 * {stride, iteration, n_correspondences, cost, inlier_rmse}.
 * pt_iters (may be NULL): device counter += executed source-point-iterations
 * (the roofline work unit).  One launch; each pair runs on one
 * CTA of 256 threads for throughput batches; latency mode (RK_ICP_WIDE=0
 * disables it) runs a pair on a thread-block cluster of 16 / 8 / 4 / 2 CTAs
 * when the batch fits one wave of such clusters (RK_ICP_CLUSTER=0|2|4|8|16
 * forces), else on one wide CTA when the batch has <= 1 / <= 2 pairs per SM
 * (1024 / 512 threads; 512 / 256 in RK_MATH_NP).  Pair indices are checked
 * on the device against cfg->n_src_images / n_dst_images (RK_ICP_BAD_PAIR). */
int rk_register_batch(const rk_sensor* s, const float* src_range, const float* dst_range,
                      const float* dst_surfel, const int32_t* pair_src,
                      const int32_t* pair_dst, int32_t batch, const double* init12,
                      const rk_icp_config* cfg, double* out12, int32_t* status,
                      int32_t* n_iters, double* stats, int32_t stats_stride,
                      unsigned long long* pt_iters, void* stream);

/* diagnostic: how many thread-block clusters of cl (2, 4, 8, 16) K3 CTAs the
 * launcher assumes co-resident for the math mode (the occupancy query it uses
 * to pick the latency tier); -1 when unavailable */
int rk_icp_cluster_capacity(int math, int cl);

/* float64 helpers of the non-bulk registration API (registration.py:96-234):
 * pts @ R.T + t; single=False association given moved points and their
 * rk_project_f64 projection; float64 robust normal equations (out29 =
 * 21 H-upper, 6 b, sum(1/w-1), sum r^2; work >= 64*29 doubles); point-to-plane
 * residuals; centroid difference mean(dst) - mean(src) (work >= 384 doubles). */
int rk_transform_points(const double* pose12, const double* pts, int64_t n, double* out,
                        void* stream);
int rk_associate_f64(const rk_sensor* s, const double* moved, const double* u, const int32_t* v,
                     const int8_t* status, int64_t n, const float* dst_surfel, double max_dist,
                     int32_t stride, uint8_t* keep, double* target, double* normal, void* stream);
int rk_normal_equations_f64(const double* pose12, const double* src, const double* tgt,
                            const double* nrm, int64_t n, double kernel, double* out29,
                            double* work, void* stream);
int rk_point_to_plane_residuals(const double* pose12, const double* src, const double* tgt,
                                const double* nrm, int64_t n, double* out, void* stream);
int rk_centroid_translation(const double* src, int64_t ns, const double* dst, int64_t nd,
                            double* out3, double* work, void* stream);

/* ------------------------------------------------------------ TSDF grid
 * VoxelBlockGrid  sdf_volume.py:35-61 : 16^3 blocks of {tsdf, weight} float32
 * pairs in a device pool, keyed through an open-addressing hash. */
int rk_grid_create(double voxel_size, double truncation, float max_weight,
                   int32_t integrate_free_space, int64_t capacity_blocks, rk_grid** out);
int rk_grid_destroy(rk_grid* g);
/* drop every block, keep the allocation (asynchronous) */
int rk_grid_clear(rk_grid* g, void* stream);
/* grow the pool / hash to hold at least capacity_blocks (synchronous) */
int rk_grid_reserve(rk_grid* g, int64_t capacity_blocks, void* stream);
/* counters (synchronous): n_blocks, capacity, overflowed-flag, last touched count */
int rk_grid_info(rk_grid* g, int64_t* out4_host, void* stream);

/* activate_blocks  sdf_volume.py:82-113 for world points (n,3) float64.
 * Resets this frame's touched list first; overflow -> rk_grid_info()[2]. */
int rk_grid_activate_points(rk_grid* g, const double* pts, int64_t n, double radius,
                            void* stream);
/* integrate_cloud_frame's activation  sdf_volume.py:198-208: to_point_cloud
 * (clip) -> pose.apply -> activate_blocks, fused; pose12 = frame->world. */
int rk_grid_activate_image(rk_grid* g, const rk_sensor* s, const float* range,
                           const double* pose12, double radius, float clip_min,
                           float clip_max, void* stream);
/* replace this frame's touched list with explicit keys (n,3) int32 (integrate(frame_keys)) */
int rk_grid_set_touched(rk_grid* g, const int32_t* keys, int64_t n, void* stream);
/* integrate  sdf_volume.py:116-186 over the current touched list.
 * inv12 = inverse pose (world->frame) formed on the host like the reference.
 * updated: device int64 accumulator (may be NULL). */
int rk_grid_integrate(rk_grid* g, const rk_sensor* s, const float* range,
                      const double* inv12, float clip_min, float clip_max, int math,
                      int64_t* updated, void* stream);
/* integrate_cloud_frame over F posed frames (sdf_volume.py:198-210 in a
 * loop, cli.py:267-283): frames (F,H,W), poses12 / invs12 (F,12) frame->world
 * and world->frame.  The activation of frame f+1 runs on an internal stream
 * while frame f integrates (two touched-set slots); safe under stream capture.
 * Afterwards the touched set is the last frame's. */
int rk_grid_integrate_frames(rk_grid* g, const rk_sensor* s, const float* frames, int32_t n_frames,
                             const double* poses12, const double* invs12, double radius,
                             float clip_min, float clip_max, int math, int64_t* updated,
                             void* stream);
/* Batched form of the sharded sequence: activate F frames into touched-set
 * slots 0..F-1 (rk_grid_reserve_slots(g, F) first), export their {count, max
 * key} pairs (F,2), all-reduce them across ranks in ONE collective (sum,
 * max), then integrate all F frames with those global pairs (NULL = local). */
int rk_grid_reserve_slots(rk_grid* g, int32_t n, void* stream);
int rk_grid_activate_frames(rk_grid* g, const rk_sensor* s, const float* frames, int32_t n_frames,
                            const double* poses12, double radius, float clip_min, float clip_max,
                            void* stream);
int rk_grid_touch_stats_frames(rk_grid* g, int32_t n_frames, int64_t* out2n, void* stream);
int rk_grid_integrate_activated(rk_grid* g, const rk_sensor* s, const float* frames,
                                int32_t n_frames, const double* invs12, const int64_t* global2n,
                                float clip_min, float clip_max, int math, int64_t* updated,
                                void* stream);
/* multi-GPU hash sharding: the grid only allocates blocks whose
 * owner(key) == rank; rk_block_owner is the host mirror of owner() for
 * keys_host (n,3).  Sharded integration needs the frame's global touched
 * count and largest key (the reference's sorted-chunk order): export the
 * local pair with rk_grid_touch_stats, all-reduce (sum, max) across ranks and
 * hand the device int64[2] back with rk_grid_set_global_touch (NULL = local). */
int rk_grid_set_shard(rk_grid* g, int32_t rank, int32_t world);
int rk_block_owner(const int32_t* keys_host, int64_t n, int32_t world, int32_t* owner_host);
int rk_grid_touch_stats(rk_grid* g, int64_t* out2, void* stream);
int rk_grid_set_global_touch(rk_grid* g, const int64_t* in2);
/* export keys (n,3) int32 of every stored block, or of the touched list */
int rk_grid_keys(rk_grid* g, int touched_only, int32_t* keys_out, int64_t cap,
                 int64_t* n_host, void* stream);
/* read / write whole blocks: vox = (n, 4096, 2) float32 {tsdf, weight} */
int rk_grid_read_blocks(rk_grid* g, const int32_t* keys, int64_t n, float* vox,
                        uint8_t* found, void* stream);
int rk_grid_write_blocks(rk_grid* g, const int32_t* keys, int64_t n, const float* vox,
                         void* stream);
/* query_sdf_many  sdf_volume.py:221-265 */
int rk_grid_query(rk_grid* g, const double* pts, int64_t n, double* sdf, double* weight,
                  uint8_t* observed, void* stream);

/* ------------------------------------------------------------ marching cubes
 * extract_mesh  mesh_extract.py:85-209 over every stored block.  tri_table:
 * device (256,16) int8 TRI_TABLE (mc_tables.py:114).  The mesh lives in the
 * grid's grow-only scratch: valid until the next rk_mc_extract on that grid
 * (copy it out with rk_mesh_copy); rk_mesh_free releases the handle only.
 * counts = {vertices, triangles}. */
typedef struct rk_mesh rk_mesh;
int rk_mc_extract(rk_grid* g, const int8_t* tri_table, float min_weight, rk_mesh** out,
                  void* stream);
int rk_mesh_info(rk_mesh* m, int64_t* counts_host);
int rk_mesh_copy(rk_mesh* m, double* verts, double* normals, int32_t* tris, void* stream);
int rk_mesh_free(rk_mesh* m);

/* ------------------------------------------------------------ synthetic input
 * render_scene (synth.py:108-134) on the device: prims = (n_prims, 16) float64
 * rows {type(0 plane,1 sphere,2 box), params...}; poses12 (B,12); out (B,H,W). */
int rk_render(const rk_sensor* s, const double* prims, int32_t n_prims,
              const double* poses12, int32_t batch, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RKB200_H */

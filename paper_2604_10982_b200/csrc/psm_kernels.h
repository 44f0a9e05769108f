// psm_kernels.h — launcher declarations of the render pipeline (K1..K7).
#ifndef PSM_KERNELS_H
#define PSM_KERNELS_H

#include <cstdint>
#include <cuda_runtime.h>

#include "psm_device.cuh"

namespace psm {

// Per-pixel contributor lists (list_cap entries per pixel). Full blending with features
// keeps them pixel-major (entry m of pixel p at p * cap + m: the feature phase reads one
// pixel's run back to back). The backward cache keeps them block-major: pixels grouped in
// the blend's 8x4 blocks, each block's lists entry-major (the 32 pixels' entry m side by
// side, entry m of a pixel at base + 32 m), so the lanes of a warp, which own one block
// and advance through their lists at similar rates, store (and the backward loads) a few
// 256 B runs instead of 32 rows a list apart (C3 cache forward 1.91 -> 1.08 ms).
__host__ __device__ inline int64_t psm_list_index(int x, int y, int width, int cap, int m) {
  const int64_t block = static_cast<int64_t>(y >> 2) * ((width + 7) >> 3) + (x >> 3);
  return (block * cap + m) * 32 + ((y & 3) * 8 + (x & 7));
}
// entries a W x H frame's lists occupy in either layout (whole blocks)
__host__ __device__ inline int64_t psm_list_slots(int width, int height, int cap) {
  return static_cast<int64_t>((width + 7) >> 3) * ((height + 3) >> 2) * 32 * cap;
}

struct BlendParams {
  const int32_t* ranges;  // [tiles][2]
  const uint32_t* vals;   // tile-sorted source ids
  const uint8_t* masks;   // beside vals: warp-block live masks (bit b: block b may be reached)
  const SurfRec* recs;
  const float* feat;      // [N][feat_dims]: f_sem | labels, fp32
  int32_t feat_dims, c_sem, n_q;
  int32_t width, height, tiles_x;
  int32_t tile_base;      // first tile of this launch (row bands)
  int32_t n_tiles;        // tiles of this launch (set by launch_blend)
  int32_t* work;          // zeroed work counter of this launch: (tile, 8x4 block) items taken
  const int32_t* order;   // optional: tile of the i-th item group (heaviest first), else tile_base + i
  double cam_cx, cam_cy, cam_fx, cam_fy;
  double chi2, alpha_min, t_min, bg0, bg1, bg2;
  int32_t support_cutoff, render_depth_normal, k_sel;
  float *color, *depth, *normal, *sem_feat, *ins_dist, *alpha_acc;
  int32_t *ins_argmax, *blend_count;
  unsigned long long* blended_total;
  int32_t* topk_dbg;      // optional [W*H*k_sel]
  uint2* lists;           // full blending with features: [W*H][list_cap]; backward cache: psm_list_index
  int32_t list_cap;
  int32_t* list_overflow;
  // panoptic epilogue (render_panoptic, metrics.cpp:339-369): when pan_ids != NULL the
  // feature phase accumulates feat64 in fp64 in blend order and writes these planes
  const double* feat64;   // [N][feat_dims] fp64
  double* lists_w;        // full blending: fp64 weights beside `lists`
  int32_t *pan_ids, *pan_classes, *pan_sem;
  // render with labels (N_q > 0): the fp64 feature phase writes sem_feat / ins_dist /
  // ins_argmax from feat64, so ins_argmax is the reference's exactly
  int32_t planes64;
  const int32_t* query_class;
  int32_t n_query_class;
  // backward cache (RenderCache::pixels, raster.cpp:399-403): when lists_t != NULL the
  // lists hold every contributor's list position with the transmittance before it, and
  // topk_pos [W*H][k_sel] the selected positions (Top-K)
  double* lists_t;
  int32_t* topk_pos;
};

// render backward (pipeline.cpp:347-486), backward.cu
struct BackwardParams {
  int32_t width, height, k_sel, topk, list_cap, c_sem, n_q;
  double cam_cx, cam_cy, cam_fx, cam_fy, bg0, bg1, bg2;
  const uint2* lists;
  const double* lists_t;
  const int32_t* topk_pos;
  const int32_t* blend_count;
  const uint32_t* vals;
  const SurfRec* recs;
  const double* surfels;   // [N][13]
  const double* feat64;    // [N][c_sem + n_q] or NULL (then feat32)
  const float* feat32;
  const double *g_color, *g_sem, *g_ins;  // upstream plane gradients (device), may be NULL
  double *d_opacity, *d_color, *d_fsem, *d_lab, *d_hinv;  // [N], [N][3], [N][c_sem], [N][n_q], [N][9]
};
void launch_pixel_backward(const BackwardParams& p, cudaStream_t st);
void launch_geom_backward(const double* surfels, const SurfRec* recs, const int32_t* valid, int64_t n,
                          const DevCamera& cam, const double* d_hinv, double* d_center, double* d_rot,
                          double* d_scales, cudaStream_t st);

// assign_labels (panoptic.cpp:36-91), labels.cu
struct LabelParams {
  int64_t n;
  int32_t c_sem, n_q, d_in, c_ins, n_alive;
  const double* surfels;     // [N][13]
  const double* f_ins;       // [N][c_ins]
  const float* feat_in;      // old rows [N][d_in] (f_sem columns first)
  const double* feat64_in;   // may be NULL
  float* feat_out;           // new rows [N][c_sem + n_q]
  double* feat64_out;        // may be NULL
  const double *q_feat, *q_mean, *q_inv;  // alive queries: [a][c_ins], [a][3], [a][9] column-major
  const int32_t* alive_index;  // alive slot -> query
  const int32_t* alive_slot;   // query -> alive slot or -1
  double* scratch;           // [n_alive][N]
  double* dist;              // optional [N][n_q]
  int32_t* argmax;           // optional [N]
};
void launch_assign_labels(const LabelParams& p, cudaStream_t st);

// K1 preprocess.cu
void launch_frame_init(unsigned long long* small, int32_t* ranges, int n_ranges, uint32_t* tcounts, int n_counts,
                       unsigned long long* dminmax, cudaStream_t stream);
void launch_preprocess(const double* surfels13, int64_t n, const DevCamera& cam, const DevRaster& rs, SurfRec* recs,
                       BinRec* bins, uint64_t* depth_bits, uint32_t* tile_counts, int32_t* valid,
                       uint32_t* n_proj, unsigned long long* depth_minmax, int32_t* err, cudaStream_t stream);

// binning.cu
void launch_tile_scan(const uint32_t* tile_counts, int tiles, uint32_t cap, int32_t* ranges, uint32_t* cursor,
                      uint32_t* totals, uint32_t* tile_start, uint32_t* rn_dev, uint32_t* rn_eff,
                      unsigned long long* nonempty, int32_t* overflow, int32_t* classes, cudaStream_t st);
void launch_emit(const int32_t* valid, int64_t n, const SurfRec* recs, const BinRec* bins, const DevRaster& rs,
                 int img_h, uint32_t* cursor, const uint32_t* tile_start, uint32_t cap, uint64_t* tile_keys,
                 const uint64_t* depth_bits, const unsigned long long* depth_minmax, int src_bits, int img_w,
                 cudaStream_t st);
void launch_sort_tiles(const int32_t* ranges, int tiles, uint64_t* tile_keys, uint64_t* key_scratch, uint32_t* tile_vals,
                       uint8_t* tile_masks, const uint64_t* depth_bits, const unsigned long long* depth_minmax,
                       int src_bits, const int32_t* classes, cudaStream_t st, cudaStream_t side, cudaStream_t side2,
                       cudaEvent_t fork, cudaEvent_t join, cudaEvent_t join2);
void launch_compact(const int32_t* valid, const int32_t* pos, const uint64_t* depth_bits, int64_t n,
                    uint64_t* keys_out, uint32_t* src_out, cudaStream_t st);
void launch_rank_of(const uint32_t* src_by_rank, const uint32_t* n_proj_dev, int64_t cap, int32_t* rank_of,
                    cudaStream_t st);
void launch_debug_keys(const int32_t* ranges, int tiles, const uint32_t* sorted_vals, const int32_t* rank_of,
                       uint64_t* keys_out, cudaStream_t st);

// scan.cu
size_t scan_cta_words(int64_t cap);
void exclusive_scan_i32(const int32_t* in, int64_t n, uint32_t* out, uint32_t* total_dev, uint32_t* cta_sums,
                        cudaStream_t st);
void exclusive_scan_u32_dev(const uint32_t* in, const uint32_t* n_dev, int64_t cap, uint32_t* out, uint32_t* total_dev,
                            uint32_t* cta_sums, cudaStream_t st);

// radix_sort.cu
size_t radix_hist_words(int64_t cap);
void radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                    int64_t cap, int begin_bit, int end_bit, uint32_t* hist, uint32_t* totals, cudaStream_t st,
                    bool* result_in_alt);
void radix_sort_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                    int64_t cap, int begin_bit, int end_bit, uint32_t* hist, uint32_t* totals, cudaStream_t st,
                    bool* result_in_alt);

// stages.cu: RenderCache outputs (psm_render_cache)
void launch_cache_pixels(const uint2* lists, int list_cap, const int32_t* cnt, const int64_t* offs,
                         const uint32_t* vals, const SurfRec* recs, const uint32_t* proj_of, int width, int height,
                         double cx, double cy, double fx, double fy, psm_contribution* out, cudaStream_t st);
void launch_cache_projected(const double* s13, int64_t n, const DevCamera& cam, double chi2, const int32_t* valid,
                            const uint32_t* proj_of, psm_projected* out, cudaStream_t st);
void launch_gather_proj(const uint32_t* vals, const uint32_t* proj_of, int64_t n, int32_t* out, cudaStream_t st);

// blend.cu
int blend_kmax_for(int k_sel);
int blend_nch_for(int feat_dims);
void launch_blend(const BlendParams& p, int tiles, bool topk, cudaStream_t st);

}  // namespace psm

#endif  // PSM_KERNELS_H

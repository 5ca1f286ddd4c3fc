/*
 * lw_oracle.h -- CPU restatement oracle for the lumenwave light-transport hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1705_01263_b200/,
 * include/, liblw_b200.so) links, imports or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, and only as the checker or the CPU baseline.
 *
 * Pinning: QMC, pixel filter, octahedral and traversal functions are checked
 * bit-exactly against the reference's own Cython kernels compiled from
 * /root/reference by oracle/Makefile (oracle/_ref/) and against golden
 * vectors generated from the reference (tests/golden/, tests/gen_golden.py).
 * The render path (lwo_render) restates SPEC.md (the reference has no
 * renderer); it and the GPU are pinned to SPEC's known answers by
 * tests/test_known_answers.py (BSDF / MIS / light and environment pdfs,
 * estimator equivalence, an independent brute-force integrator).
 */
#pragma once
#include <stdint.h>
#include "../include/lw_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* _kernels.py:160-222 */
double lwo_halton_dim(const int64_t* bases, const int64_t* perm_flat, const int64_t* perm_offset,
                      int64_t dim, int64_t index);
void lwo_halton_batch(const int64_t* bases, const int64_t* perm_flat, const int64_t* perm_offset,
                      int64_t dim, const int64_t* indices, int64_t n, double* out);

/* _kernels.py:87-134 */
double lwo_gauss_filter_offset(double u);
void lwo_pixel_offset_batch(const double* u, int64_t n, double* out);

/* _kernels.py:233-342 */
int64_t lwo_oct_encode(double x, double y, double z);
void lwo_oct_decode(int64_t packed, double* out3);
void lwo_oct_roundtrip_batch(const double* vecs, int64_t n, double* out);

/* _kernels.py:357-585.  mode: LW_TRAVERSE_COMPAT | LW_TRAVERSE_CORRECTED | LW_TRAVERSE_BRUTE */
void lwo_intersect_batch(int mode, const double* bounds, const int64_t* children, const int64_t* order,
                         const double* verts, int64_t ntris, const double* origins, const double* dirs,
                         const double* tmaxs, int64_t n, double* out_t, int64_t* out_tri, double* out_bary);

/* geometry.py:100-148.  Returns node count; arrays must hold 2*ntris-1 (>=1) nodes. */
int64_t lwo_build_bvh(const double* verts, int64_t ntris, double* bounds, int64_t* children, int64_t* order);

/* Vose alias table. prob/alias/pdf have n entries. Returns 0 on success. */
int lwo_alias_build(const double* weights, int64_t n, double* prob, int32_t* alias, double* pdf);

/* Closest hit / any hit in the render traversal order (near-first, conservative cull). */
typedef struct lwo_scene lwo_scene;
lwo_scene* lwo_scene_create(const lw_scene_desc* desc);
void lwo_scene_destroy(lwo_scene* s);
void lwo_trace_closest_batch(const lwo_scene* s, const double* origins, const double* dirs, const double* tmaxs,
                             int64_t n, double* out_t, int64_t* out_tri, double* out_bary);
void lwo_trace_any_batch(const lwo_scene* s, const double* origins, const double* dirs, const double* tmaxs,
                         int64_t n, int32_t* out_occluded);
void lwo_camera_rays(const lwo_scene* s, const lw_render_params* p, const int64_t* sample_index, int64_t n,
                     double* out_o, double* out_d);
/* Progressive render of pixels [pix_begin, pix_end) x iterations [it_begin, it_end) into fb (int64 W*H*3). */
void lwo_render(const lwo_scene* s, const lw_render_params* p, int64_t pix_begin, int64_t pix_end,
                int64_t it_begin, int64_t it_end, int64_t* fb, int nthreads, lw_render_stats* stats);

/* Light hierarchy (device: lw_lighttree.cuh).  Node record =
 * lo[3] hi[3] tot flux[8] as 15 doubles + right child (or -(emitter+1) at a leaf).
 * lwo_light_tree: node count (0 when the scene uses the alias table); copies when outputs given. */
int64_t lwo_light_tree(const lwo_scene* s, double* nodes15, int32_t* right, uint64_t* path, int32_t* depth);
/* sample_light from points x with unit normals nrm and uniforms u: emitter, selection probability,
 * rescaled uniform.  light_pdf: selection probability of emitter e from (x, nrm). */
void lwo_light_sample_batch(const lwo_scene* s, const double* x, const double* nrm, const double* u, int64_t n,
                            int64_t* out_e, double* out_psel, double* out_u);
void lwo_light_pdf_batch(const lwo_scene* s, const int64_t* e, const double* x, const double* nrm, int64_t n,
                         double* out_psel);

/* Environment pyramid (device: lw_envpyr.cuh).  info: 1 if built (levels out).
 * sample: base texel index, its probability and the in-texel (u, v) for octahedral-packed normals
 * and uniforms uv [n,2].  pdf: probability of texel for the packed normal. */
int lwo_env_pyramid_info(const lwo_scene* s, int32_t* nlevels);
void lwo_env_sample_batch(const lwo_scene* s, const int64_t* packed_normal, const double* uv, int64_t n,
                          int64_t* out_texel, double* out_p, double* out_uv);
void lwo_env_pdf_batch(const lwo_scene* s, const int64_t* packed_normal, const int64_t* texel, int64_t n,
                       double* out_p);

/* lwo_render plus light-path-expression layers: product-DFA tables from
 * lpe.compile_layers; layer_fb holds nlayers int64 framebuffers of W*H*3. */
void lwo_render_lpe(const lwo_scene* s, const lw_render_params* p, int64_t pix_begin, int64_t pix_end,
                    int64_t it_begin, int64_t it_end, int64_t* fb, int nlayers, int nstates, const int16_t* trans,
                    const uint8_t* accept, int start, int64_t* layer_fb, int nthreads, lw_render_stats* stats);

/* Known-answer surface of the render math (same semantics as the lw_bsdf_eval_batch /
 * lw_bsdf_sample_batch / lw_ctx_nee_light_sample / lw_ctx_emission_pdf entries of the library). */
void lwo_bsdf_eval_batch(const lw_material* m, const double* wo, const double* wi, int64_t n, double* out_f,
                         double* out_pdf);
void lwo_bsdf_sample_batch(const lw_material* m, const double* wo, const int32_t* front, const double* uv, int64_t n,
                           double* out_wi, double* out_weight, double* out_pdf, int32_t* out_flags);
void lwo_nee_light_sample_batch(const lwo_scene* s, const double* p, const double* ngf, const double* uv, int64_t n,
                                double* out_wi, double* out_le, double* out_pdf, double* out_tmax, int64_t* out_e);
void lwo_emission_pdf_batch(const lwo_scene* s, const double* o, const double* d, const int32_t* nprev, int64_t n,
                            double* out_le, double* out_pdf, int64_t* out_e);

/* Deterministic math shared by oracle and device (restated independently in lw_detmath.cuh). */
void lwo_sincos2pi(double u, double* s, double* c);
double lwo_atan2(double y, double x);

#ifdef __cplusplus
}
#endif

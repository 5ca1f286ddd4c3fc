/*
 * lw_b200.h -- C ABI of liblw_b200.so, the B200 (sm_100a) light-transport hot path.
 *
 * Drop-in boundary for the reference package `lumenwave` (arXiv 1705.01263):
 * every stateless entry point replaces one function of the Cython kernel module
 * `lumenwave.core._kernels` selected at `lumenwave/core/__init__.py:9-11`, with
 * the same argument meaning (caller-owned C-contiguous float64/int64 buffers,
 * misses encoded as data, no exceptions from the kernels).  The render entry
 * points implement the SPEC-only call stack `cmd_render`
 * -> scheduler -> wavefront -> integrator
 * (SPEC.md:366-506), which the reference declares but does not ship.
 *
 * Conventions
 *  - Every function returns LW_OK (0) or an LW_ERR_* code; lw_last_error()
 *    returns a thread-local message for the last failure.  Device faults are
 *    reported as LW_ERR_CUDA, never as aborts.
 *  - Pointers without a `_device` suffix are HOST pointers; the library copies
 *    in and out.  `*_device` variants take device pointers and run on the
 *    context's stream (or the per-thread default stream for stateless calls).
 *  - No torch/Python types cross this boundary.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LW_ABI_VERSION 1

/* status codes */
#define LW_OK 0
#define LW_ERR_INVALID 1   /* bad argument (the reference wrappers raise ValueError) */
#define LW_ERR_CUDA 2      /* CUDA runtime / kernel failure */
#define LW_ERR_NOMEM 3     /* device allocation failed */
#define LW_ERR_STATE 4     /* call order violated (e.g. render before scene upload) */
#define LW_ERR_OVERFLOW 5  /* sample index exceeds 64 bits (qmc.py:194-195 OverflowError) */

/* traversal semantics for lw_intersect_batch (_kernels.py:422-585) */
#define LW_TRAVERSE_COMPAT 0    /* bit-exact replica of the pristine reference, defects D1/D2 included */
#define LW_TRAVERSE_CORRECTED 1 /* D1 (permuted origin) and D2 (on-face zero-direction slabs) fixed, LIFO order */
#define LW_TRAVERSE_BRUTE 2     /* corrected triangle test over every triangle, min (t, id) */

/* wavefront stage tags (_kernels.py:42-48) */
#define LW_STAGE_GENERATE 0
#define LW_STAGE_TRACE 1
#define LW_STAGE_MATERIAL 2
#define LW_STAGE_NEE 3
#define LW_STAGE_ENVMATTE 4
#define LW_STAGE_TERMINATED 5
#define LW_STAGE_COUNT 6

/* elemental BSDFs (sceneformat.py:223 BSDF_KINDS) */
#define LW_BSDF_DIFFUSE 0
#define LW_BSDF_GLOSSY 1
#define LW_BSDF_SPECULAR_REFLECT 2
#define LW_BSDF_SPECULAR_TRANSMIT 3
#define LW_MAX_LAYERS 4 /* sceneformat.py:225 */

/* light-path-expression events (paper_1705_01263_b200/lpe.py) */
#define LW_EV_C 0  /* camera */
#define LW_EV_RD 1 /* diffuse reflection */
#define LW_EV_RG 2 /* glossy reflection */
#define LW_EV_RS 3 /* specular reflection */
#define LW_EV_TS 4 /* specular transmission */
#define LW_EV_L 5  /* emissive triangle */
#define LW_EV_E 6  /* environment */
#define LW_EV_COUNT 7

/* environment kinds (sceneformat.py:304-309) */
#define LW_ENV_NONE 0
#define LW_ENV_CONSTANT 1
#define LW_ENV_IMAGE 2 /* lat-long, row 0 = +y pole */

/* execution engines */
#define LW_ENGINE_WAVEFRONT 0
#define LW_ENGINE_MEGAKERNEL 1

typedef struct lw_layer {
  int32_t kind;      /* LW_BSDF_* */
  int32_t coat;      /* Fresnel-weighted coating (Layer.coat, sceneformat.py:243) */
  double tint[3];    /* Layer.tint constant node value */
  double weight;     /* Layer.weight constant node value (scalar) */
  double roughness;  /* GGX alpha for glossy layers */
} lw_layer;

typedef struct lw_material {
  int32_t nlayers;
  int32_t thin_walled;
  lw_layer layers[LW_MAX_LAYERS];
  double ior; /* Material.ior (sceneformat.py:256) */
} lw_material;

typedef struct lw_scene_desc {
  /* flattened world-space triangle soup (geometry.py:23-32, flatten_instances 58-97) */
  int64_t ntris;
  const double* verts;       /* [ntris, 9] p0 p1 p2 */
  const double* normals;     /* [ntris, 9] per-vertex shading normals */
  const int32_t* material;   /* [ntris] material index */
  int32_t nmaterials;
  int32_t env_kind;          /* LW_ENV_* */
  const lw_material* materials;
  /* emissive triangles (sceneformat.py:285-293 Emitter; Material.emission) */
  int64_t nemit;
  const int64_t* emit_tri;       /* [nemit] global triangle id */
  const double* emit_radiance;   /* [nemit, 3] */
  const int32_t* emit_twosided;  /* [nemit] */
  const double* emit_weight;     /* [nemit] light-selection weight (luminance(L) * area) */
  /* environment (sceneformat.py:304-309) */
  double env_constant[3];
  double env_scale;
  int32_t env_width, env_height;
  const float* env_image;        /* [env_height, env_width, 3] radiance */
  const double* env_weight;      /* [env_height * env_width] luminance * sin(theta_center) */
  double p_env;                  /* probability of choosing the environment in NEE */
  /* camera (sceneformat.py:333-340, block_camera 776-801) */
  double cam_pos[3];
  double cam_fwd[3];
  double cam_right[3];
  double cam_up[3];
  double tan_half_fov; /* tan(fov_y / 2), computed by the host */
  int32_t bvh_kind;    /* render BVH: LW_BVH_SAH (default) or LW_BVH_MEDIAN (the reference's tree) */
  int32_t light_sampler; /* NEE light selection flags: 0 = LW_LIGHTS_ALIAS (flat alias tables over
                            emitter and texel weights); | LW_LIGHTS_TREE: light hierarchy over the
                            emitters; | LW_LIGHTS_ENV_PYRAMID: environment pyramid
                            with normal-binned top levels */
} lw_scene_desc;

#define LW_LIGHTS_ALIAS 0
#define LW_LIGHTS_TREE 1
#define LW_LIGHTS_ENV_PYRAMID 2

#define LW_BVH_SAH 0    /* binned SAH, breadth-first */
#define LW_BVH_MEDIAN 1 /* geometry.py:100-148 median split (built on the GPU) */

typedef struct lw_render_params {
  int32_t width;
  int32_t height;
  int32_t max_depth;    /* path segments traced from the camera */
  int32_t rr_start;     /* first bounce index with Russian roulette (4) */
  /* DimensionTable arrays (qmc.py:274-305) */
  int64_t ndims;
  const int64_t* bases;
  const int64_t* perm_flat;
  int64_t perm_len;
  const int64_t* perm_offset;
  /* engine knobs */
  int32_t engine;            /* LW_ENGINE_* */
  int32_t pool_log2;         /* wavefront state pool = 2^pool_log2 slots */
  double regen_fraction;     /* regenerate when free slots exceed this fraction of the pool (paper: 0.5) */
  int64_t megakernel_tail;   /* switch to the megakernel once active paths drop below this (0 = never) */
  int32_t estimator;         /* LW_EST_*: how emitter / environment radiance is estimated */
  int32_t compact_state;     /* 1: compressed path state: ray directions as 2x16-bit
                                octahedral codes (the reference codec, _kernels.py:233-299), throughput,
                                radiance and BSDF pdf in FP32 -- quantised where produced, identically in
                                both engines and the oracle; 0: FP64 state */
} lw_render_params;

/* estimators (SPEC.md:400-402 estimator equivalence): balance-heuristic MIS of light sampling and
 * BSDF sampling (the renderer), light sampling only (NEE weight 1; emitters / environment reached by
 * BSDF sampling after a non-specular vertex count 0), BSDF sampling only (no NEE; every emitter /
 * environment hit counts with weight 1).  All three are unbiased estimators of the same image. */
#define LW_EST_MIS 0
#define LW_EST_NEE 1
#define LW_EST_BSDF 2

typedef struct lw_render_stats {
  int64_t paths;          /* (pixel, iteration) samples completed */
  int64_t rays_extension; /* closest-hit rays traced */
  int64_t rays_shadow;    /* any-hit rays traced */
  int64_t waves;          /* wavefront stage rounds executed */
  int64_t regenerations;  /* regeneration events */
  int64_t nonfinite;      /* samples whose radiance was non-finite (accumulated as 0) */
} lw_render_stats;

/* per-kernel profile of the last pass (lw_ctx_set_instrumentation) */
typedef struct lw_kernel_profile {
  double trace_ext_ms;       /* summed CUDA-event time of the extension-ray trace kernel launches */
  double trace_shadow_ms;    /* same for the shadow-ray trace kernel */
  double total_ms;           /* whole pass */
  int64_t trace_ext_launches;
  int64_t trace_shadow_launches;
  int64_t kernel_launches;   /* every kernel this library launched in the pass */
  int64_t ext_rays, ext_nodes, ext_tris;        /* traversal work (LW_INSTR_COUNT) */
  int64_t shadow_rays, shadow_nodes, shadow_tris;
  /* per wavefront stage (LW_INSTR_TIME): summed CUDA-event time and launches, index LW_PROF_* */
  double stage_ms[6];
  int64_t stage_launches[6];
  int64_t pool_slots;        /* wavefront pool of the pass */
  int64_t waves;             /* stage rounds */
  int64_t paths;             /* paths generated and flushed */
  int64_t shadow_unoccluded; /* shadow rays that added their NEE contribution */
} lw_kernel_profile;

#define LW_PROF_GENERATE 0     /* k_generate: flush + regenerate + extension queue */
#define LW_PROF_TRACE_EXT 1    /* k_trace_ext(_p): closest hit */
#define LW_PROF_SHADE_NEE 2    /* k_shade_nee: light sample, BSDF eval, shadow-ray setup */
#define LW_PROF_SHADE 3        /* k_shade: emission/MIS, BSDF sampling, roulette, next ray */
#define LW_PROF_TRACE_SHADOW 4 /* k_trace_shadow(_p): any hit + NEE accumulation */
#define LW_PROF_OTHER 5        /* wave bookkeeping (k_wave_begin / k_wave_end, tail) */
#define LW_PROF_END 6

#define LW_INSTR_TIME 1  /* bracket trace launches with CUDA events */
#define LW_INSTR_COUNT 2 /* count node visits / triangle tests (separate kernel instantiation) */

/* fixed-point framebuffer: per pixel 3 x int64 in units of 2^-LW_FB_FRAC_BITS radiance */
#define LW_FB_FRAC_BITS 20
#define LW_FB_SAMPLE_CLAMP 4294967296.0 /* 2^32: per-sample radiance clamp before quantisation */

/* ---- library ---------------------------------------------------------------------- */
const char* lw_last_error(void);
int lw_abi_version(void);
int lw_device_count(int* count);
int lw_set_device(int device);

/* ---- stateless kernels (reference kernel-module surface) ------------------------- */

/* halton_batch (_kernels.py:211-222): out[i] = scrambled radical inverse of indices[i] in dim */
int lw_halton_batch(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                    const int64_t* perm_offset, int64_t dim, const int64_t* indices, int64_t n, double* out);
int lw_halton_batch_device(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                           const int64_t* perm_offset, int64_t dim, const int64_t* indices_device, int64_t n,
                           double* out_device);

/* sample_pixel_offset (_kernels.py:132-134), batched: u [n,2] -> out [n,2] */
int lw_pixel_offset_batch(const double* u, int64_t n, double* out);

/* oct_roundtrip_batch (_kernels.py:321-342), compress/decompress (302-318) batched */
int lw_oct_roundtrip_batch(const double* vecs, int64_t n, double* out);
int lw_oct_encode_batch(const double* vecs, int64_t n, int64_t* out);
int lw_oct_decode_batch(const int64_t* packed, int64_t n, double* out);

/* intersect_batch (_kernels.py:548-585).  `instances` of the reference is unused and omitted. */
int lw_intersect_batch(int mode, const double* bounds, const int64_t* children, int64_t nnodes,
                       const int64_t* order, const double* verts, int64_t ntris, const double* origins,
                       const double* dirs, const double* tmaxs, int64_t n, double* out_t, int64_t* out_tri,
                       double* out_bary);
int lw_intersect_batch_device(int mode, const double* bounds, const int64_t* children, int64_t nnodes,
                              const int64_t* order, const double* verts, int64_t ntris, const double* origins,
                              const double* dirs, const double* tmaxs, int64_t n, double* out_t,
                              int64_t* out_tri, double* out_bary);

/* build_bvh (geometry.py:100-148) on the GPU; same arrays as the reference.
 * bounds [2*ntris-1 (>=1), 6], children [.., 2], order [ntris]; *nnodes receives the node count. */
int lw_bvh_build(const double* verts, int64_t ntris, double* bounds, int64_t* children, int64_t* order,
                 int64_t* nnodes);

/* Vose alias table over non-negative weights (host; shared by light and environment selection) */
int lw_alias_build(const double* weights, int64_t n, double* prob, int32_t* alias, double* pdf);

/* ---- render context (one per GPU, owned by one host thread) --------------------- */
typedef struct lw_ctx lw_ctx;
int lw_ctx_create(int device, lw_ctx** out);
int lw_ctx_destroy(lw_ctx* ctx);
/* run all work of this context on an external stream (cudaStream_t; NULL = the context's own) */
int lw_ctx_set_stream(lw_ctx* ctx, void* stream);
int lw_ctx_set_instrumentation(lw_ctx* ctx, int flags);
int lw_ctx_kernel_profile(lw_ctx* ctx, lw_kernel_profile* out);
/* uploads geometry, builds the BVH on the device, builds light/env alias tables */
int lw_scene_upload(lw_ctx* ctx, const lw_scene_desc* scene);
int lw_render_configure(lw_ctx* ctx, const lw_render_params* params);
/* clears the fixed-point framebuffer */
int lw_framebuffer_clear(lw_ctx* ctx);
/* renders every pixel for iterations [it_begin, it_end) into the framebuffer.  Asynchronous: the
 * wavefront runs as one CUDA-graph launch whose conditional WHILE node repeats the wave until no
 * work is left and no path is alive (device-side termination), so the call returns once the pass
 * is queued on the context's stream; passes, reduces and accumulations queue behind each other.
 * Statistics / profiles are completed on demand (lw_get_stats, lw_ctx_kernel_profile,
 * lw_ctx_synchronize), which is also where device faults of the pass are reported.  The
 * megakernel tail switch (megakernel_tail > 0) and LW_GRAPH=0 use a host-driven loop instead. */
int lw_render_pass(lw_ctx* ctx, int64_t it_begin, int64_t it_end);
/* renders pixels [pix_begin, pix_end) only (parity subsets) */
int lw_render_pass_pixels(lw_ctx* ctx, int64_t it_begin, int64_t it_end, int64_t pix_begin, int64_t pix_end);
int lw_ctx_synchronize(lw_ctx* ctx);
int lw_framebuffer_download(lw_ctx* ctx, int64_t* host_fb);           /* W*H*3 int64 */
int lw_framebuffer_resolve(lw_ctx* ctx, double inv_samples, float* host_rgb); /* W*H*3 float32 */
int lw_framebuffer_copy_device(lw_ctx* ctx, void* dst_device);         /* D2D copy for NCCL reduction */
int lw_framebuffer_load_device(lw_ctx* ctx, const void* src_device);   /* D2D copy back after reduction */
int lw_framebuffer_upload(lw_ctx* ctx, const int64_t* host_fb);       /* H2D: resume from a checkpoint */
/* Progressive accumulation on the context's stream (asynchronous): dst_device (W*H*3 int64,
 * 16-byte aligned, caller-owned) += framebuffer; clear != 0 also zeroes the framebuffer for the
 * next pass.  One kernel instead of copy + add + clear. */
int lw_framebuffer_accumulate(lw_ctx* ctx, void* dst_device, int clear);

/* Sample-space partition across GPUs: one context per GPU and
 * process; every rank renders a disjoint block of iterations, then the pass framebuffers are
 * sum-reduced in place with an NCCL all-reduce on the context's stream (int64 addition is
 * associative: the image is bit-identical for any rank count).  NCCL is loaded at first use
 * (libnccl.so.2).  lw_comm_unique_id: rank 0 creates the id, the caller broadcasts it (e.g. over
 * torch.distributed); lw_ctx_comm_init: every rank joins; lw_framebuffer_reduce: asynchronous
 * all-reduce of the framebuffer (and LPE layer framebuffers). */
#define LW_COMM_ID_BYTES 128
int lw_comm_unique_id(uint8_t* id_out);
int lw_ctx_comm_init(lw_ctx* ctx, const uint8_t* id, int rank, int world);
int lw_framebuffer_reduce(lw_ctx* ctx);
int lw_get_stats(lw_ctx* ctx, lw_render_stats* stats);
/* debug/parity surface of the render traversal (near-first, conservative cull) */
int lw_ctx_trace_closest(lw_ctx* ctx, const double* origins, const double* dirs, const double* tmaxs, int64_t n,
                         double* out_t, int64_t* out_tri, double* out_bary);
int lw_ctx_trace_any(lw_ctx* ctx, const double* origins, const double* dirs, const double* tmaxs, int64_t n,
                     int32_t* out_occluded);
int lw_ctx_camera_rays(lw_ctx* ctx, const int64_t* sample_index, int64_t n, double* out_o, double* out_d);
/* Light hierarchy of the uploaded scene (LW_LIGHTS_TREE; PAPER.md:215-253, SPEC.md:196-221
 * LightHierarchy / sample_light / light_pdf).  info: node count (0 = alias-table selection).
 * download: nodes as 15 doubles (lo[3] hi[3] tot flux[8]) + right child (leaf: -(emitter+1)),
 * per-emitter branch bits and depth (-1 = weight 0, not in the tree).  sample: emitter, selection
 * probability and rescaled uniform for points x with unit normals nrm.  pdf: selection
 * probability of emitter e from (x, nrm), the MIS counterpart of sample. */
int lw_ctx_light_tree_info(lw_ctx* ctx, int64_t* nnodes);
int lw_ctx_light_tree_download(lw_ctx* ctx, double* nodes15, int32_t* right, uint64_t* path, int32_t* depth);
int lw_ctx_light_sample(lw_ctx* ctx, const double* x, const double* nrm, const double* u, int64_t n,
                        int64_t* out_e, double* out_psel, double* out_u);
int lw_ctx_light_pdf(lw_ctx* ctx, const int64_t* e, const double* x, const double* nrm, int64_t n,
                     double* out_psel);
/* Environment pyramid (LW_LIGHTS_ENV_PYRAMID; PAPER.md:262-276, SPEC.md:222-230 sample_env /
 * env_pdf): levels (0 = not built).  sample: base texel index (row * width + col), its probability
 * and the in-texel (u, v) for octahedral-packed facing normals and uniforms uv [n,2]; pdf: texel
 * probability for the packed normal. */
/* Light path expressions: the product automaton of lpe.compile_layers
 * (trans [nstates, LW_EV_COUNT], per-state accepting-layer bit mask, start state).  While set, the
 * renderer routes every radiance contribution to the layers whose expression accepts the
 * contribution's event string (int64 fixed-point layer framebuffers, cleared with the main one);
 * nlayers = 0 removes the layers.  Both engines route (the stage kernels' LPE instantiations). */
int lw_ctx_set_lpe(lw_ctx* ctx, int32_t nlayers, int32_t nstates, const int16_t* trans, const uint8_t* accept,
                   int32_t start);
int lw_ctx_lpe_download(lw_ctx* ctx, int32_t layer, int64_t* fb);
/* H2D copy of one layer framebuffer (checkpoint resume of a render with layers) */
int lw_ctx_lpe_upload(lw_ctx* ctx, int32_t layer, const int64_t* fb);
int lw_ctx_env_pyramid_info(lw_ctx* ctx, int32_t* nlevels);
int lw_ctx_env_sample(lw_ctx* ctx, const int64_t* packed_normal, const double* uv, int64_t n, int64_t* out_texel,
                      double* out_p, double* out_uv);
int lw_ctx_env_pdf(lw_ctx* ctx, const int64_t* packed_normal, const int64_t* texel, int64_t n, double* out_p);
/* Known-answer surface of the render math (SPEC.md:309-317 bsdf_evaluate / bsdf_sample,
 * 394-402 next_event + MIS, 204-230 sample_light / light_pdf / sample_env / env_pdf), the same
 * device functions the engines run.
 * lw_bsdf_eval_batch: f (RGB) and pdf (solid angle, non-delta lobes) for local-frame directions
 *   (z = shading normal), layer weights from wo.z.
 * lw_bsdf_sample_batch: sampled wi, weight f*cos/pdf (delta lobes: the lobe's throughput), pdf
 *   (0 for delta lobes) and flags: bit 0 sampled, bit 1 delta, bit 2 transmission, bits 8+ the
 *   LPE event (LW_EV_*).  front: the ray arrived on the front side (transmission eta).
 * lw_mis_weight_batch: the balance heuristic a / (a + b) of the engines.
 * lw_ctx_nee_light_sample: the light half of NEE at points p with facing normals ngf for NEE
 *   uniforms uv: direction, radiance, solid-angle pdf (0: no light), shadow-ray tmax, emitter
 *   (-1 = environment).
 * lw_ctx_emission_pdf: what BSDF sampling meets along (o, d): radiance and the light-sampling pdf
 *   MIS weighs it against (nprev: packed facing normal of the vertex the ray leaves), emitter
 *   (-1 environment, -2 non-emissive surface). */
int lw_bsdf_eval_batch(const lw_material* m, const double* wo, const double* wi, int64_t n, double* out_f,
                       double* out_pdf);
int lw_bsdf_sample_batch(const lw_material* m, const double* wo, const int32_t* front, const double* uv, int64_t n,
                         double* out_wi, double* out_weight, double* out_pdf, int32_t* out_flags);
int lw_mis_weight_batch(const double* pdf_a, const double* pdf_b, int64_t n, double* out);
int lw_ctx_nee_light_sample(lw_ctx* ctx, const double* p, const double* ngf, const double* uv, int64_t n,
                            double* out_wi, double* out_le, double* out_pdf, double* out_tmax, int64_t* out_emitter);
int lw_ctx_emission_pdf(lw_ctx* ctx, const double* o, const double* d, const int32_t* nprev, int64_t n,
                        double* out_le, double* out_pdf, int64_t* out_emitter);
/* BVH arrays the context built (reference layout), for parity checks */
int lw_ctx_bvh_info(lw_ctx* ctx, int64_t* nnodes);
int lw_ctx_bvh_download(lw_ctx* ctx, double* bounds, int64_t* children, int64_t* order);
/* kernel timing of the last pass: milliseconds spent in trace kernels and total (CUDA events) */
int lw_ctx_last_pass_timing(lw_ctx* ctx, double* trace_ms, double* total_ms, int64_t* kernel_launches);

#ifdef __cplusplus
}
#endif

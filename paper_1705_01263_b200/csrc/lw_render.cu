// lw_render.cu -- render context, scene upload and the two execution engines.
//
// SPEC.md:508-588 (wavefront) and PAPER.md:599-699:
//  * sample states live in a fixed-size SoA pool (one array per field, coalesced);
//  * each wave runs the stage kernels generate/regenerate -> trace -> material+NEE ->
//    shadow trace over compact queues rebuilt every stage with warp ballots
//    (__ballot_sync + __popc, one atomic per warp);
//  * terminated slots are regenerated with new (iteration, pixel) work once more than
//    `regen_fraction` of the pool is free (paper: one half);
//  * the tail of a pass can switch to the megakernel.
// Radiance is accumulated per path into an int64 fixed-point framebuffer, so the image is
// independent of execution strategy, pool size, switch threshold and GPU count.
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <vector>

#include <cub/cub.cuh>

#include "lw_common.cuh"
#include "lw_host.h"
#include "lw_integrator.cuh"

using namespace lw;

// occupancy knobs (min resident blocks of 128 threads per SM) for the FP64-heavy stage kernels
// persistent trace kernels: refill when >= LW_REFILL lanes of a warp are idle; speculative
// traversal in the persistent kernels (LW_SPEC) and in the one-ray-per-thread kernels (LW_SPEC_SMEM)
#ifndef LW_REFILL
#define LW_REFILL 24
#endif
#ifndef LW_SPEC
#define LW_SPEC 3  // bit 0: extension rays, bit 1: shadow rays
#endif
#ifndef LW_SPEC_SMEM
#define LW_SPEC_SMEM 2  // bit 0: extension rays (C2 trace +2 %: off), bit 1: shadow rays
#endif
#ifndef LW_TRACE_MINB
#define LW_TRACE_MINB 8
#endif
#ifndef LW_SHADOW_MINB
#define LW_SHADOW_MINB 8
#endif
#ifndef LW_SHADE_MINB
#define LW_SHADE_MINB 4
#endif
#ifndef LW_NEE_MINB
#define LW_NEE_MINB 4
#endif
// k_generate: 4 blocks of 256 -> 64 registers (5 -> 48 with spills: 1-3 % slower generate; no
// bound -> 90 registers: C2 generate 0.22 -> 0.31 ms)
#ifndef LW_SHADE_PREFETCH
#define LW_SHADE_PREFETCH 2  // shading kernels: 1 queue entries read a grid stride ahead, 2 + NEE hit / flags
#endif
#ifndef LW_SHADE_K2
#define LW_SHADE_K2 1  // k_shade (diffuse classes): also the next entry's hit record a stride ahead
#endif
#ifndef LW_NEE_L2
#define LW_NEE_L2 1  // k_shade_nee also instantiated for the two-layer classes
#endif
#ifndef LW_GEN_PREFETCH
#define LW_GEN_PREFETCH 2  // 0 none, 1 stage bytes two rounds ahead, 2 + flush data one round ahead
#endif
#ifndef LW_GEN_MINB
#define LW_GEN_MINB 4
#endif
// the same for the diffuse material class (LW_MC_DIFFUSE instantiations, fewer live registers)
#ifndef LW_SHADE_MINB_D
#define LW_SHADE_MINB_D 4
#endif
#ifndef LW_NEE_MINB_D
#define LW_NEE_MINB_D 4
#endif

namespace {

struct WorkRange {
  long long it_begin, nits, pix_begin, npix;
  long long tiles_x;  // > 0: whole frame enumerated in tiles of tw x th pixels x ti iterations (32 items)
  int tw, th, ti;
};

struct Counters {
  WorkRange wr;  // the pass's work (read by k_generate / the wave condition: graph launches stay valid)
  int gwaves, overflow;  // waves run by the CUDA-graph loop; set if it hit the wave limit
  int stamp_n;           // LW_INSTR_TIME: stage timestamps written this pass
  unsigned long long work_next;  // next work item (iteration-major over the pixel range)
  int n_ext, n_shadow, n_alive;
  int regen_now;  // decision of the current wave's regeneration step
  unsigned long long n_alive_ull;
  unsigned long long rays_ext, rays_shadow, paths, nonfinite, regens, waves;
  unsigned long long ext_nodes, ext_tris, sh_nodes, sh_tris;
  unsigned long long sh_unocc;  // shadow rays that reached their light (NEE contribution added)
  int ext_next, sh_next;  // queue heads of the persistent trace kernels
  // tail queue: once the pool is mostly empty the last compacted extension queue is
  // kept for the rest of the pass (no more compaction); stage kernels skip its finished entries
  int tail, tail_armed, n_trace;
};

// SoA of 16-byte vectors: slot s of every array is one LDG.128/STG.128, and a warp's 32
// consecutive slots cover 512 contiguous bytes per array
struct Pool {
  int size = 0;
  double2 *ray0, *ray1, *ray2;  // (o.x, o.y) (o.z, d.x) (d.y, d.z)
  double2 *tp0, *tp1, *tp2;     // (beta.x, beta.y) (beta.z, L.x) (L.y, L.z)
  double2* misc;                // (pdf_prev, sample index bits)
  double2 *hit0, *hit1;         // (t, bu) (bv, tri bits)
  double2 *sh0, *sh1, *sh2, *sh3, *sh4;  // shadow (o.x,o.y) (o.z,d.x) (d.y,d.z) (tmax,c.x) (c.y,c.z)
  int* pix;
  int* flags;  // bounce | spec_prev << 8
  int* nprev;  // octahedral-packed facing normal of the previous vertex (light-tree MIS)
  // light-path-expression layers (only touched by the LPE instantiations of the stage kernels)
  int* lpe_state;            // automaton state of the path
  double2 *sh5, *sh6, *sh7;  // NEE contribution split: (d.x, d.y) (d.z, g.x) (g.y, g.z)
  int* sh_lpe;               // automaton state at the NEE vertex | terminal event << 16
  unsigned char* stage;  // LW_STAGE_GENERATE / TRACE / TERMINATED
  int *q_ext, *q_shadow;
  void* block = nullptr;
};

// everything a wave's launches depend on (the CUDA graph is rebuilt when it changes)
struct WaveCfg {
  int pool = 0, cmp = 0, lpe_on = 0, ltm = 0, use_smem = 0, count = 0, timed = 0, persist_mask = 0, tail_div = 0, mc = 0;
  size_t smem = 0, ltsm = 0;
  void* pool_block = nullptr;
  long long epoch = -1;
  bool operator==(const WaveCfg& o) const {
    return pool == o.pool && cmp == o.cmp && lpe_on == o.lpe_on && ltm == o.ltm && use_smem == o.use_smem &&
           count == o.count && timed == o.timed && persist_mask == o.persist_mask && tail_div == o.tail_div && mc == o.mc &&
           smem == o.smem && ltsm == o.ltsm && pool_block == o.pool_block && epoch == o.epoch;
  }
};

constexpr int kStampCap = 1 << 16;  // stage timestamps per pass (7 per wave)
// per-context device / pinned block: Counters, running statistics, stage timestamps
constexpr size_t kAccOff = (sizeof(Counters) + 63) / 64 * 64;
constexpr size_t kStampOff = kAccOff + 64;
constexpr size_t kCtrBytes = kStampOff + sizeof(unsigned long long) * kStampCap;

}  // namespace

struct lw_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool has_scene = false, configured = false;
  DevScene S;
  std::vector<void*> scene_allocs;
  DeviceBVH ref_bvh;
  bool ref_built = false;
  int64_t lt_nodes = 0;  // light hierarchy nodes (0 = alias-table light selection)
  std::vector<LwLightNode> lt_dfs;  // the hierarchy as built (depth-first), for lw_ctx_light_tree_download
  std::vector<unsigned long long> lt_path;
  std::vector<int> lt_depth;
  LwLpe lpe = {nullptr, nullptr, 0, 0, nullptr, 0};  // light-path-expression layers (megakernel)
  int64_t ntris = 0;
  lw_render_params params;
  QmcDim* d_qdims = nullptr;
  uint16_t* d_qperm = nullptr;
  unsigned long long* d_fb = nullptr;
  int64_t fb_pixels = 0;
  Pool pool;
  Counters* d_cnt = nullptr;
  Counters* h_cnt = nullptr;  // pinned mirror
  lw_render_stats stats;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_total_ms = 0.0, last_trace_ms = 0.0;
  int64_t last_launches = 0;
  size_t smem_bytes = 0;  // scene bytes staged in shared memory (0 = use global/L1)
  size_t pool_bytes = 0;  // bytes of pool.block
  // persistent lane-refill trace kernels (with speculative traversal): bits 0 / 1 extension /
  // shadow rays on global-memory BVHs, bits 2 / 3 the same on shared-memory BVHs; all on by
  // default (C2 +4 %, C3 +13 %); LW_TRACE_PERSIST=<mask> overrides (A/B measurements)
  int persist_mask = getenv("LW_TRACE_PERSIST") ? atoi(getenv("LW_TRACE_PERSIST")) : 15;
  bool persist = (persist_mask & 1) != 0;
  bool persist_sh = (persist_mask & 2) != 0;
  // tail queue: keep the compacted queue once fewer than pool / tail_div paths are
  // alive and nothing is left to regenerate (0 = compact every wave); LW_TAIL_QUEUE overrides
  int tail_div = getenv("LW_TAIL_QUEUE") ? atoi(getenv("LW_TAIL_QUEUE")) : 16;
  // scene class (LW_MC_* in lw_integrator.cuh) the shading kernels are instantiated for:
  // mat_diffuse = every material one uncoated diffuse layer (set by lw_scene_upload); the
  // environment / light-selection bits come from DevScene.  LW_MATCLASS=0 forces LW_MC_ANY (A/B).
  bool mat_diffuse = false;
  int mat_max_layers = LW_MAX_LAYERS;  // largest layer count of the scene's materials
  bool mat_class_on = getenv("LW_MATCLASS") ? atoi(getenv("LW_MATCLASS")) != 0 : true;
  int nrnodes = 0;        // internal nodes of the render BVH
  cudaStream_t own_stream = nullptr;
  int instr = 0;
  std::vector<cudaEvent_t> evpool;  // pairs bracketing trace launches
  lw_kernel_profile prof;
  ncclComm_t comm = nullptr;  // sample-space partition: per-pass framebuffer sum over the ranks
  int comm_rank = 0, comm_world = 1;
  // CUDA-graph wave loop (device-side termination) and asynchronous pass bookkeeping
  bool use_graph = getenv("LW_GRAPH") ? atoi(getenv("LW_GRAPH")) != 0 : true;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t side_stream = nullptr;  // scene-upload copies overlapping the BVH build
  cudaEvent_t ev_side0 = nullptr, ev_side1 = nullptr;
  cudaGraphExec_t wave_exec = nullptr;
  WaveCfg wave_key;
  WaveCfg last_key;  // configuration of the previous wavefront pass
  long long epoch = 0;  // bumped by scene upload / configure / LPE changes (parameters baked into the graph)
  bool pass_pending = false, pass_graph = false, pass_timed = false;
  int64_t pass_host_launches = 0;
  unsigned long long *d_acc = nullptr, *h_acc = nullptr;        // running statistics [6]
  unsigned long long *d_stamps = nullptr, *h_stamps = nullptr;  // stage timestamps of the pass
};

void free_lpe(lw_ctx* c) {
  if (c->lpe.trans) cudaFreeAsync((void*)c->lpe.trans, c->stream);
  if (c->lpe.accept) cudaFreeAsync((void*)c->lpe.accept, c->stream);
  if (c->lpe.fb) cudaFreeAsync(c->lpe.fb, c->stream);
  c->lpe = LwLpe{nullptr, nullptr, 0, 0, nullptr, 0};
}

namespace {

template <class T>
int dev_upload(lw_ctx* c, T*& dst, const T* src, int64_t count) {
  LW_CUDA_TRY(cudaMallocAsync(&dst, sizeof(T) * (count > 0 ? count : 1), c->stream));
  c->scene_allocs.push_back(dst);
  if (count > 0) LW_CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyHostToDevice, c->stream));
  return LW_OK;
}

template <class T>
int dev_alloc(lw_ctx* c, T*& dst, int64_t count) {
  LW_CUDA_TRY(cudaMallocAsync(&dst, sizeof(T) * (count > 0 ? count : 1), c->stream));
  c->scene_allocs.push_back(dst);
  return LW_OK;
}

void free_scene(lw_ctx* c) {
  for (void* p : c->scene_allocs) cudaFreeAsync(p, c->stream);
  c->scene_allocs.clear();
  if (c->ref_bvh.bounds) cudaFreeAsync(c->ref_bvh.bounds, c->stream);
  if (c->ref_bvh.children) cudaFreeAsync(c->ref_bvh.children, c->stream);
  if (c->ref_bvh.order) cudaFreeAsync(c->ref_bvh.order, c->stream);
  c->ref_bvh = DeviceBVH();
  c->ref_built = false;
  c->lt_nodes = 0;
  c->has_scene = false;
}

// Per-device cache of wavefront-pool blocks (several GB): a destroyed context hands its block to
// the next one instead of returning it to the stream-ordered allocator, where interleaved scene
// and BVH-build allocations fragment the address range and force a fresh multi-GB mapping
// (measured: C3 end-to-end 79 vs 198 Mpaths/s with a 2^24-slot pool).
struct PoolBlock {
  int device;
  size_t bytes;
  void* p;
};
std::mutex g_pool_mu;
std::vector<PoolBlock> g_pool_free;
constexpr size_t kPoolCache = 2;

void free_pool(lw_ctx* c) {
  if (c->pool.block) {
    cudaStreamSynchronize(c->stream);  // the block may still be in use by queued kernels
    bool kept = false;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      if (g_pool_free.size() < kPoolCache) {
        g_pool_free.push_back({c->device, c->pool_bytes, c->pool.block});
        kept = true;
      }
    }
    if (!kept) cudaFree(c->pool.block);
  }
  c->pool = Pool();
  c->pool_bytes = 0;
}

void* take_pool_block(int device, size_t bytes, size_t& got) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (size_t k = 0; k < g_pool_free.size(); k++)
    if (g_pool_free[k].device == device && g_pool_free[k].bytes >= bytes && g_pool_free[k].bytes <= 2 * bytes) {
      void* p = g_pool_free[k].p;
      got = g_pool_free[k].bytes;
      g_pool_free.erase(g_pool_free.begin() + k);
      return p;
    }
  return nullptr;
}

// ---- warp-aggregated queue append ---------------------------------------------------------
// all 32 lanes of the warp must call it (kernels keep grid-stride loops warp-uniform)
__device__ __forceinline__ int warp_push(int* count, bool pred) {
  unsigned m = __ballot_sync(0xffffffffu, pred);
  if (m == 0) return -1;
  int lane = threadIdx.x & 31;
  int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!pred) return -1;
  return base + __popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ void warp_add(unsigned long long* ctr, unsigned long long v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, v);
}

// stage the render BVH in shared memory when it fits (small scenes: Cornell box); nodes are laid
// out with an LW_SNODE-byte stride (RenderBVH::nstride): with 144 bytes, lanes reading the same
// field of different nodes hit different banks instead of the same four
#ifndef LW_SNODE
#define LW_SNODE 144
#endif
__host__ __device__ __forceinline__ size_t smem_bvh_bytes(long long nnodes, long long ntris) {
  return (size_t)nnodes * LW_SNODE + (size_t)ntris * sizeof(LTri);
}

__device__ __forceinline__ RenderBVH stage_bvh(const RenderBVH& g, int nnodes, unsigned char* smem, bool use_smem) {
  if (!use_smem) return g;
  const int4* src = reinterpret_cast<const int4*>(g.nodes);
  const int per = (int)(sizeof(WNode) / 16), sper = LW_SNODE / 16;
  int4* dst = reinterpret_cast<int4*>(smem);
  for (int k = threadIdx.x; k < nnodes * per; k += blockDim.x) dst[(k / per) * sper + k % per] = src[k];
  LTri* st = reinterpret_cast<LTri*>(smem + (size_t)nnodes * LW_SNODE);
  src = reinterpret_cast<const int4*>(g.tris);
  dst = reinterpret_cast<int4*>(st);
  int nt4 = (int)g.ntris * (int)(sizeof(LTri) / 16);
  for (int k = threadIdx.x; k < nt4; k += blockDim.x) dst[k] = src[k];
  __syncthreads();
  RenderBVH b = g;
  b.nodes = reinterpret_cast<const WNode*>(smem);
  b.nstride = LW_SNODE;
  b.tris = st;
  return b;
}

// ---- scene preparation kernels ------------------------------------------------------------

__global__ void k_internal_flags(const long long* __restrict__ children, long long nnodes, int* __restrict__ flag) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < nnodes) flag[k] = children[2 * k] >= 0 ? 1 : 0;
}

__host__ __device__ __forceinline__ int leaf_ref(long long start, long long count) { return (int)(-(1 + ((start << 3) | count))); }

__global__ void k_build_rnodes(const double* __restrict__ bounds, const long long* __restrict__ children,
                               long long nnodes, const int* __restrict__ imap, SahNode* __restrict__ out) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= nnodes) return;
  if (children[2 * k] < 0) return;
  SahNode r;
#pragma unroll
  for (int c = 0; c < 2; c++) {
    long long ch = children[2 * k + c];
#pragma unroll
    for (int a = 0; a < 6; a++) r.box[6 * c + a] = bounds[6 * ch + a];
    long long c0 = children[2 * ch], c1 = children[2 * ch + 1];
    r.ref[c] = c0 >= 0 ? imap[ch] : leaf_ref(-(c0 + 1), c1);
  }
  out[imap[k]] = r;
}

__global__ void k_build_ltris(const double* __restrict__ verts, const long long* __restrict__ order, long long n,
                              LTri* __restrict__ out) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  long long t = order[j];
  LTri r;
#pragma unroll
  for (int k = 0; k < 9; k++) r.v[k] = verts[9 * t + k];
  r.id = t;
  out[j] = r;
}

// ---- binary -> 4-wide collapse (level-synchronous over the binary tree) -------------------
//
// A wide node is rooted at a binary node and takes its two children; while it has fewer than
// four, the internal child with the largest surface area (first on ties) is replaced by its two
// children.  Wide nodes keep the id of their binary root (the array is sparse, parents before
// children as in the binary numbering).  need[] tracks the traversal stack depth a path can
// reach (sum of children-1 over the wide nodes above), so the upload can reject trees deeper
// than the fixed traversal stack instead of overflowing it.

__device__ __forceinline__ double sah_area12(const double* b) {
  double dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
  return (dx * dy + dy * dz) + dz * dx;
}

__global__ void k_collapse_level(const SahNode* __restrict__ bin, const int* __restrict__ fin, const int* __restrict__ nin,
                                 int* __restrict__ fout, int* __restrict__ nout, int* __restrict__ need,
                                 WNode* __restrict__ out, int* __restrict__ max_need) {
  int n = *nin;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int b = fin[i];
    int cref[4];
    double cbox[4][6];
    const SahNode& nb = bin[b];
#pragma unroll
    for (int c = 0; c < 2; c++) {
      cref[c] = nb.ref[c];
#pragma unroll
      for (int a = 0; a < 6; a++) cbox[c][a] = nb.box[6 * c + a];
    }
    int k = 2;
    while (k < 4) {
      int sel = -1;
      double sa = -1.0;
      for (int j = 0; j < k; j++) {
        if (cref[j] < 0) continue;
        double ar = sah_area12(cbox[j]);
        if (ar > sa) {
          sa = ar;
          sel = j;
        }
      }
      if (sel < 0) break;
      const SahNode& e = bin[cref[sel]];
      cref[sel] = e.ref[0];
      cref[k] = e.ref[1];
      for (int a = 0; a < 6; a++) {
        cbox[sel][a] = e.box[a];
        cbox[k][a] = e.box[6 + a];
      }
      k++;
    }
    WNode w;
    float lo[3][4], hi[3][4];
    int rr[4];
    for (int c = 0; c < 4; c++) {
      bool v = c < k;
      rr[c] = v ? cref[c] : LW_REF_NONE;
      for (int a = 0; a < 3; a++) {
        lo[a][c] = v ? __double2float_rd(cbox[c][a]) : INFINITY;
        hi[a][c] = v ? __double2float_ru(cbox[c][3 + a]) : -INFINITY;
      }
    }
    for (int a = 0; a < 3; a++) {
      w.lo[a] = make_float4(lo[a][0], lo[a][1], lo[a][2], lo[a][3]);
      w.hi[a] = make_float4(hi[a][0], hi[a][1], hi[a][2], hi[a][3]);
    }
    w.ref = make_int4(rr[0], rr[1], rr[2], rr[3]);
    w.pad = make_int4(k, 0, 0, 0);
    out[b] = w;
    int nd = need[b] + (k - 1);
    atomicMax(max_need, nd);
    for (int c = 0; c < k; c++) {
      if (cref[c] < 0) continue;
      need[cref[c]] = nd;
      fout[atomicAdd(nout, 1)] = cref[c];
    }
  }
}

__global__ void k_build_ltris_i32(const double* __restrict__ verts, const int* __restrict__ order, long long n,
                                  LTri* __restrict__ out) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  long long t = order[j];
  LTri r;
#pragma unroll
  for (int k = 0; k < 9; k++) r.v[k] = verts[9 * t + k];
  r.id = t;
  out[j] = r;
}

__global__ void k_emitters(const double* __restrict__ verts, const long long* __restrict__ emit_tri, long long nemit,
                           double* __restrict__ area, int* __restrict__ emit_of_tri) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nemit) return;
  const double* v = verts + 9 * emit_tri[e];
  double e1x = v[3] - v[0], e1y = v[4] - v[1], e1z = v[5] - v[2];
  double e2x = v[6] - v[0], e2y = v[7] - v[1], e2z = v[8] - v[2];
  double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
  area[e] = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
  emit_of_tri[emit_tri[e]] = (int)e;
}

// ---- environment alias tables, built on the GPU at upload -----------------------------------
// Two-level Vose tables over the texel weights (oracle: env_alias2_build): one thread per row runs
// the host alias_build (lw_capi.cu) op for op over the row -- scaled weights kept in `prob` in
// place, worklists in global scratch -- then one thread builds the table over the row sums and a
// grid multiplies the per-texel pdfs by their row's probability.  Replaces a sequential host Vose
// over W*H texels (~0.1-0.3 s for 4096x2048) and its 168 MB pageable upload.
__global__ void k_env_rows(const double* __restrict__ w, int W, int H, double* __restrict__ prob,
                           int* __restrict__ alias, double* __restrict__ pdf, double* __restrict__ rsum,
                           int* __restrict__ sstk, int* __restrict__ lstk) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= H) return;
  const size_t o = (size_t)r * W;
  const double* wr = w + o;
  double* pr = prob + o;
  int* ar = alias + o;
  double* dr = pdf + o;
  int* small = sstk + o;
  int* large = lstk + o;
  double total = 0.0;
  bool ok = true;
  for (int c = 0; c < W; c++) {
    double x = wr[c];
    if (!(x >= 0.0) || x == INFINITY) ok = false;
    total += x;
  }
  rsum[r] = total;
  if (!ok || !(total > 0.0)) {  // a row without weight is never drawn
    for (int c = 0; c < W; c++) {
      pr[c] = 1.0;
      ar[c] = c;
      dr[c] = 0.0;
    }
    return;
  }
  int ns = 0, nl = 0;
  const double dn = (double)W;
  for (int c = 0; c < W; c++) {
    double pc = wr[c] / total;
    dr[c] = pc;
    double sc = pc * dn;
    pr[c] = sc;
    if (sc < 1.0)
      small[ns++] = c;
    else
      large[nl++] = c;
  }
  while (ns > 0 && nl > 0) {
    int sm = small[--ns];
    int l = large[--nl];
    ar[sm] = l;  // prob[sm] keeps its scaled weight
    double nv = (pr[l] + pr[sm]) - 1.0;
    pr[l] = nv;
    if (nv < 1.0)
      small[ns++] = l;
    else
      large[nl++] = l;
  }
  while (nl > 0) {
    int l = large[--nl];
    pr[l] = 1.0;
    ar[l] = l;
  }
  while (ns > 0) {
    int sm = small[--ns];
    pr[sm] = 1.0;
    ar[sm] = sm;
  }
}

// the table over the row sums (one thread; H entries); *bad = 1 if the sums are not valid weights
__global__ void k_env_marginal(const double* __restrict__ rsum, int H, double* __restrict__ rprob,
                               int* __restrict__ ralias, double* __restrict__ rpdf, int* __restrict__ sstk,
                               int* __restrict__ lstk, int* __restrict__ bad) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double total = 0.0;
  for (int r = 0; r < H; r++) {
    double x = rsum[r];
    if (!(x >= 0.0) || x == INFINITY) {
      *bad = 1;
      return;
    }
    total += x;
  }
  if (!(total > 0.0)) {
    *bad = 1;
    return;
  }
  *bad = 0;
  int ns = 0, nl = 0;
  const double dn = (double)H;
  for (int r = 0; r < H; r++) {
    double pc = rsum[r] / total;
    rpdf[r] = pc;
    double sc = pc * dn;
    rprob[r] = sc;
    if (sc < 1.0)
      sstk[ns++] = r;
    else
      lstk[nl++] = r;
  }
  while (ns > 0 && nl > 0) {
    int sm = sstk[--ns];
    int l = lstk[--nl];
    ralias[sm] = l;
    double nv = (rprob[l] + rprob[sm]) - 1.0;
    rprob[l] = nv;
    if (nv < 1.0)
      sstk[ns++] = l;
    else
      lstk[nl++] = l;
  }
  while (nl > 0) {
    int l = lstk[--nl];
    rprob[l] = 1.0;
    ralias[l] = l;
  }
  while (ns > 0) {
    int sm = sstk[--ns];
    rprob[sm] = 1.0;
    ralias[sm] = sm;
  }
}

// The same construction with one thread block per table, staged in shared memory (the per-thread
// form above walks W texels of its own row through L2 with dependent loads: 8.8 ms for 4096x2048,
// 64 warps on the whole GPU).  Thread 0 keeps every order-dependent step sequential -- the row sum
// in texel order and the Vose pairing -- while the block loads the weights, divides by the sum and
// sorts texels into the small / large worklists with a block scan (both in texel order, as the
// sequential pushes leave them), so every value is the sequential one.  Shared memory: W scaled
// weights (8 B) + one W-entry worklist array holding the small stack from the bottom and the large
// stack from the top (their sizes add up to at most W).
constexpr int kAliasThreads = 256;
__device__ void alias_build_block(const double* __restrict__ w, int n, double* __restrict__ prob, int* __restrict__ alias,
                                  double* __restrict__ pdf, double* total_out, int* bad_out, bool uniform_if_bad,
                                  double* sp, int* stk) {
  using BlockScan = cub::BlockScan<int, kAliasThreads>;
  __shared__ typename BlockScan::TempStorage ts;
  __shared__ double s_total;
  __shared__ int s_ok, s_carry;
  for (int c = threadIdx.x; c < n; c += kAliasThreads) sp[c] = w[c];
  __syncthreads();
  if (threadIdx.x == 0) {
    double total = 0.0;
    int ok = 1;
    for (int c = 0; c < n; c++) {
      double x = sp[c];
      if (!(x >= 0.0) || x == INFINITY) ok = 0;
      total += x;
    }
    s_total = total;
    s_ok = ok && total > 0.0;
    s_carry = 0;
    if (total_out) *total_out = total;
    if (bad_out) *bad_out = s_ok ? 0 : 1;
  }
  __syncthreads();
  const double total = s_total;
  if (!s_ok) {
    if (uniform_if_bad)  // a row without weight is never drawn
      for (int c = threadIdx.x; c < n; c += kAliasThreads) {
        prob[c] = 1.0;
        alias[c] = c;
        pdf[c] = 0.0;
      }
    return;
  }
  // scaled weights and the worklists in index order (small: sc < 1 from the bottom, large from the top)
  const double dn = (double)n;
  for (int base = 0; base < n; base += kAliasThreads) {
    int c = base + threadIdx.x;
    int small = 0;
    if (c < n) {
      double pc = sp[c] / total;
      pdf[c] = pc;
      double sc = pc * dn;
      sp[c] = sc;
      small = sc < 1.0 ? 1 : 0;
    }
    int pos, cnt;
    BlockScan(ts).ExclusiveSum(small, pos, cnt);
    int carry = s_carry;
    if (c < n) {
      if (small)
        stk[carry + pos] = c;
      else
        stk[n - 1 - (c - carry - pos)] = c;  // large entry k = c - (smalls before c) at n-1-k
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + cnt;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int ns = s_carry, nl = n - ns;
    while (ns > 0 && nl > 0) {
      int sm = stk[--ns];
      int l = stk[n - nl];
      --nl;
      alias[sm] = l;  // prob[sm] keeps its scaled weight
      double nv = (sp[l] + sp[sm]) - 1.0;
      sp[l] = nv;
      if (nv < 1.0)
        stk[ns++] = l;
      else
        stk[n - 1 - nl++] = l;
    }
    while (nl > 0) {
      int l = stk[n - nl];
      --nl;
      sp[l] = 1.0;
      alias[l] = l;
    }
    while (ns > 0) {
      int sm = stk[--ns];
      sp[sm] = 1.0;
      alias[sm] = sm;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += kAliasThreads) prob[c] = sp[c];
}

__global__ void __launch_bounds__(kAliasThreads) k_env_rows_blk(const double* __restrict__ w, int W, int H,
                                                                double* __restrict__ prob, int* __restrict__ alias,
                                                                double* __restrict__ pdf, double* __restrict__ rsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* sp = reinterpret_cast<double*>(smem);
  int* stk = reinterpret_cast<int*>(sp + W);
  for (int r = blockIdx.x; r < H; r += gridDim.x) {
    const size_t o = (size_t)r * W;
    alias_build_block(w + o, W, prob + o, alias + o, pdf + o, rsum + r, nullptr, true, sp, stk);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kAliasThreads) k_env_marginal_blk(const double* __restrict__ rsum, int H,
                                                                    double* __restrict__ rprob, int* __restrict__ ralias,
                                                                    double* __restrict__ rpdf, int* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* sp = reinterpret_cast<double*>(smem);
  int* stk = reinterpret_cast<int*>(sp + H);
  alias_build_block(rsum, H, rprob, ralias, rpdf, nullptr, bad, false, sp, stk);
}

__global__ void k_env_pdf(double* __restrict__ pdf, const double* __restrict__ rpdf, int W, long long n) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    pdf[j] = rpdf[j / W] * pdf[j];
}

// ---- megakernel ----------------------------------------------------------------------------

// work item -> (iteration, pixel) -> QMC sample index.  A whole frame is enumerated in 8x4-pixel
// tiles, so the 32 paths a warp generates (and, through the slot-ordered queues, traces and
// shades) cover a compact patch instead of a 32x1 strip; the sample index of a (pixel, iteration)
// is unchanged, so is every result.
__device__ __forceinline__ long long work_index(const DevScene& S, const WorkRange& w, long long item, int& pix) {
  long long it, p;
  if (w.tiles_x > 0) {
    // iteration block, then tile, then the 32 items of the tile (pixel-minor)
    const long long blk = item / (w.npix * w.ti), q = item % (w.npix * w.ti);
    const long long t = q >> 5;
    const int r = (int)(q & 31), tp = w.tw * w.th, ri = r / tp, rp = r % tp;
    it = w.it_begin + blk * w.ti + ri;
    p = ((t / w.tiles_x) * w.th + rp / w.tw) * (long long)S.W + (t % w.tiles_x) * w.tw + rp % w.tw;
  } else {
    it = w.it_begin + item / w.npix;
    p = w.pix_begin + item % w.npix;
  }
  pix = (int)p;
  return it * ((long long)S.W * S.H) + p;
}

template <bool CMP>
__device__ __forceinline__ void run_to_completion(const DevScene& S, const RenderBVH& bvh, PathState& ps,
                                                  unsigned long long& next, unsigned long long& nsh,
                                                  const LwLpe* lpe = nullptr, long long pix = 0) {
  for (;;) {
    double o[3] = {ps.o.x, ps.o.y, ps.o.z}, d[3] = {ps.d.x, ps.d.y, ps.d.z};
    LwHit h;
    lw_trace_closest(bvh, o, d, INFINITY, h);
    next++;
    ShadowRay sh;
    bool alive = lw_path_shade<CMP>(S, ps, h, sh, lpe, pix);
    if (sh.valid) {
      double so[3] = {sh.o.x, sh.o.y, sh.o.z}, sd[3] = {sh.d.x, sh.d.y, sh.d.z};
      nsh++;
      if (!lw_trace_any(bvh, so, sd, sh.tmax)) {
        ps.L = CMP ? lw_q32v(ps.L + sh.contrib) : ps.L + sh.contrib;
        if (lpe) {
          lw_lpe_route(lpe, lw_lpe_step(lpe, lw_lpe_step(lpe, sh.lpe, LW_EV_RD), sh.term), pix, sh.c_diffuse);
          lw_lpe_route(lpe, lw_lpe_step(lpe, lw_lpe_step(lpe, sh.lpe, LW_EV_RG), sh.term), pix, sh.c_glossy);
        }
      }
    }
    if (!alive) break;
  }
}

// LPE = true: every contribution is also routed to the light-path-expression layers
template <bool LPE, bool CMP>
__global__ void __launch_bounds__(128) k_megakernel(DevScene S, WorkRange w, unsigned long long* __restrict__ fb,
                                                    Counters* __restrict__ cnt, int nrnodes, int use_smem, LwLpe lpe) {
  extern __shared__ __align__(16) unsigned char smem[];
  RenderBVH bvh = stage_bvh(S.bvh, nrnodes, smem, use_smem != 0);
  long long total = w.nits * w.npix;
  unsigned long long next = 0, nsh = 0, bad = 0, paths = 0;
  for (long long base = blockIdx.x * (long long)blockDim.x; base < total; base += (long long)gridDim.x * blockDim.x) {
    long long item = base + threadIdx.x;
    if (item < total) {
      int pix;
      long long index = work_index(S, w, item, pix);
      PathState ps;
      lw_path_init<CMP>(S, index, ps);
      if (LPE) ps.lpe = lw_lpe_step(&lpe, lpe.start, LW_EV_C);
      run_to_completion<CMP>(S, bvh, ps, next, nsh, LPE ? &lpe : nullptr, pix);
      bad += lw_accumulate(fb, pix, ps.L);
      paths++;
    }
  }
  warp_add(&cnt->rays_ext, next);
  warp_add(&cnt->rays_shadow, nsh);
  warp_add(&cnt->nonfinite, bad);
  warp_add(&cnt->paths, paths);
}

// ---- wavefront stages -----------------------------------------------------------------------
//
// Every slot carries a stage tag (the reference's STAGE_* contract, _kernels.py:42-48):
// GENERATE = free, TRACE = extension ray ready, TERMINATED = finished path awaiting its
// framebuffer flush.  Each wave: k_wave_begin (decision) -> k_generate (pool order: flush,
// regenerate, ascending extension queue) -> k_trace_ext -> k_shade (material + NEE) ->
// k_trace_shadow.  Queues are rebuilt from the pool every wave in ascending slot order
// (SPEC.md:375), so SoA loads stay coalesced however the population fragments.

#define F_BOUNCE 0xff
#define F_SPEC (1 << 8)

// Pool layout of a path (16-byte vectors).  FP64 state: ray0 (o.x, o.y), ray1 (o.z, d.x), ray2
// (d.y, d.z), tp0 (beta.x, beta.y), tp1 (beta.z, L.x), tp2 (L.y, L.z), misc (pdf_prev, index) --
// 112 bytes.  Compact state (S.compact): ray0 (o.x, o.y), ray1 (o.z, oct(d) << 32
// | fp32 pdf_prev), tp0 as float4 (beta.xyz, L.x), tp1 (fp32 L.y | L.z << 32, index) -- 64 bytes.
__device__ __forceinline__ unsigned long long pack2f(double lo, double hi) {
  return ((unsigned long long)__float_as_uint((float)hi) << 32) | __float_as_uint((float)lo);
}

__device__ __forceinline__ void load_ray(const Pool& P, int s, double o[3], double d[3], bool compact) {
  double2 a = P.ray0[s], b = P.ray1[s];
  o[0] = a.x;
  o[1] = a.y;
  o[2] = b.x;
  if (compact) {
    v3 v = lw_oct_dir((unsigned)((unsigned long long)__double_as_longlong(b.y) >> 32));
    d[0] = v.x;
    d[1] = v.y;
    d[2] = v.z;
    return;
  }
  double2 c = P.ray2[s];
  d[0] = b.y;
  d[1] = c.x;
  d[2] = c.y;
}

// nprev (previous vertex normal) is only consumed by the light hierarchy / environment pyramid MIS
template <int MC = LW_MC_ANY>
__device__ __forceinline__ bool needs_nprev(const DevScene& S) {
  return lw_light_mode<MC>(S) != 0 || ((MC & LW_MC_NOENV) ? 0 : S.env_mode) != 0;
}

__device__ __forceinline__ void load_state(const Pool& P, int s, PathState& ps, bool nprev, bool compact) {
  double2 a = P.ray0[s], b = P.ray1[s];
  ps.o = mk3(a.x, a.y, b.x);
  if (compact) {
    unsigned long long bits = (unsigned long long)__double_as_longlong(b.y);
    ps.doct = (unsigned)(bits >> 32);
    ps.d = lw_oct_dir(ps.doct);
    ps.pdf_prev = (double)__uint_as_float((unsigned)bits);
    float4 t0 = reinterpret_cast<const float4*>(P.tp0)[s];
    double2 t1 = P.tp1[s];
    unsigned long long lb = (unsigned long long)__double_as_longlong(t1.x);
    ps.beta = mk3((double)t0.x, (double)t0.y, (double)t0.z);
    ps.L = mk3((double)t0.w, (double)__uint_as_float((unsigned)lb), (double)__uint_as_float((unsigned)(lb >> 32)));
    ps.index = __double_as_longlong(t1.y);
  } else {
    double2 c = P.ray2[s];
    ps.d = mk3(b.y, c.x, c.y);
    double2 t0 = P.tp0[s], t1 = P.tp1[s], t2 = P.tp2[s];
    ps.beta = mk3(t0.x, t0.y, t1.x);
    ps.L = mk3(t1.y, t2.x, t2.y);
    double2 m = P.misc[s];
    ps.pdf_prev = m.x;
    ps.index = __double_as_longlong(m.y);
    ps.doct = 0;
  }
  int f = P.flags[s];
  ps.bounce = f & F_BOUNCE;
  ps.spec_prev = (f & F_SPEC) ? 1 : 0;
  ps.nprev = nprev ? P.nprev[s] : 0;
}

// compact: every stored value is already FP32-representable / an oct code (quantised where produced)
__device__ __forceinline__ void store_state(const Pool& P, int s, const PathState& ps, bool nprev, bool compact) {
  P.ray0[s] = make_double2(ps.o.x, ps.o.y);
  if (compact) {
    P.ray1[s] = make_double2(ps.o.z, __longlong_as_double((long long)(((unsigned long long)ps.doct << 32) |
                                                                          __float_as_uint((float)ps.pdf_prev))));
    reinterpret_cast<float4*>(P.tp0)[s] =
        make_float4((float)ps.beta.x, (float)ps.beta.y, (float)ps.beta.z, (float)ps.L.x);
    P.tp1[s] = make_double2(__longlong_as_double((long long)pack2f(ps.L.y, ps.L.z)), __longlong_as_double(ps.index));
  } else {
    P.ray1[s] = make_double2(ps.o.z, ps.d.x);
    P.ray2[s] = make_double2(ps.d.y, ps.d.z);
    P.tp0[s] = make_double2(ps.beta.x, ps.beta.y);
    P.tp1[s] = make_double2(ps.beta.z, ps.L.x);
    P.tp2[s] = make_double2(ps.L.y, ps.L.z);
    P.misc[s] = make_double2(ps.pdf_prev, __longlong_as_double(ps.index));
  }
  P.flags[s] = ps.bounce | (ps.spec_prev ? F_SPEC : 0);
  if (nprev) P.nprev[s] = ps.nprev;
}

__device__ __forceinline__ v3 load_L(const Pool& P, int s, bool compact) {
  if (compact) {
    float lx = reinterpret_cast<const float4*>(P.tp0)[s].w;
    unsigned long long lb = (unsigned long long)__double_as_longlong(P.tp1[s].x);
    return mk3((double)lx, (double)__uint_as_float((unsigned)lb), (double)__uint_as_float((unsigned)(lb >> 32)));
  }
  double2 t1 = P.tp1[s], t2 = P.tp2[s];
  return mk3(t1.y, t2.x, t2.y);
}

// paper §3.1.3: regenerate only once more than regen_fraction of the pool is free (or nothing
// is in flight); one thread decides so every block of k_generate sees the same choice
//
// Tail queue ("when the runtime of the compaction kernel exceeds the runtime of the
// state kernel, we generate a single tail queue once"): once no work is left to regenerate and
// fewer than pool / tail_div paths are alive, the next compaction is the last; later waves reuse
// that queue (n_ext unchanged), k_generate returns at once and the stage kernels skip entries whose
// path has finished.  `force` (the final flush) leaves tail mode.
__global__ void k_wave_begin(Counters* cnt, int pool, double regen_fraction, int force, int tail_div) {
  const long long total = cnt->wr.nits * cnt->wr.npix;
  if (force) cnt->tail = cnt->tail_armed = 0;
  if (cnt->tail_armed) cnt->tail = 1;
  int alive = cnt->n_alive;
  cnt->n_shadow = 0;
  cnt->n_alive = 0;
  cnt->ext_next = 0;
  cnt->sh_next = 0;
  if (cnt->tail) {
    cnt->regen_now = 0;
    cnt->n_trace = alive;  // rays this wave (the queue also holds finished entries)
    return;
  }
  bool regen = force || (pool - alive) > (int)(regen_fraction * (double)pool) || alive == 0;
  cnt->regen_now = regen ? 1 : 0;
  if (regen) cnt->regens += 1;
  if (!force && !regen && tail_div > 0 && (long long)cnt->work_next >= total && alive < pool / tail_div)
    cnt->tail_armed = 1;  // this wave's compaction builds the tail queue
  cnt->n_ext = 0;
}

// pool order: flush TERMINATED slots, refill free slots with new (iteration, pixel) samples and
// compact TRACE slots into the extension queue.  Each WARP owns a contiguous slot range (no block
// barriers): a counting pass reads the range's stage bytes 16 at a time (one 16-byte load per
// lane) and sizes the warp's claims, which it takes with two atomics (work items, queue segment);
// the writing pass walks the range 32 slots per round (lane = slot, coalesced), assigning items
// and queue positions in slot order from ballot prefixes.  The generated samples are the first
// `granted` free slots of the range, so a lane's queue offset is trace_prefix + min(want_prefix,
// granted_left).  (Block-granular with a barrier per 256 slots, this scan cost ~170 us per wave on
// C2 even when nothing was left to do; the per-warp form is bound by the stage-byte reads.)
template <bool LPE, bool CMP>
__global__ void __launch_bounds__(256, LW_GEN_MINB) k_generate(DevScene S, Pool P, unsigned long long* __restrict__ fb,
                                                  Counters* __restrict__ cnt, LwLpe lpe) {
  if (cnt->tail) return;  // tail queue: no compaction, nothing to regenerate
  const WorkRange w = cnt->wr;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const bool regen = cnt->regen_now != 0;
  const long long total = w.nits * w.npix;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int per = (int)((((long long)P.size + nwarps * 512 - 1) / (nwarps * 512)) * 512);
  const int r0 = (int)min(gwarp * per, (long long)P.size);
  const int r1 = min(r0 + per, P.size);
  if (r0 >= r1) return;  // warp-uniform
  // pass 1: sizes of the claims (16 stage bytes per lane per load; ranges are multiples of 512)
  int c_want = 0, c_trace = 0;
  for (int s = r0 + 16 * lane; s < r1; s += 512) {
    uint4 v = *reinterpret_cast<const uint4*>(P.stage + s);
    unsigned wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 16; k++) {
      unsigned b = (wd[k >> 2] >> (8 * (k & 3))) & 0xffu;
      c_trace += b == LW_STAGE_TRACE ? 1 : 0;
      c_want += (regen && b != LW_STAGE_TRACE) ? 1 : 0;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    c_want += __shfl_xor_sync(0xffffffffu, c_want, off);
    c_trace += __shfl_xor_sync(0xffffffffu, c_trace, off);
  }
  long long wb = 0;
  int eb = 0, granted = 0;
  if (lane == 0) {
    wb = c_want ? (long long)atomicAdd(&cnt->work_next, (unsigned long long)c_want) : 0;
    long long left = total - wb;
    granted = left <= 0 ? 0 : (int)min(left, (long long)c_want);
    eb = (c_trace + granted) ? atomicAdd(&cnt->n_ext, c_trace + granted) : 0;
  }
  long long wnext = __shfl_sync(0xffffffffu, wb, 0);  // next work item of this warp
  int gleft = __shfl_sync(0xffffffffu, granted, 0);  // work items left to place
  int enext = __shfl_sync(0xffffffffu, eb, 0);       // next queue position of this warp
  unsigned long long bad = 0, paths = 0;
  if (c_trace == 0 && (!regen || c_want == 0)) return;  // nothing to flush, generate or queue here
#if LW_GEN_PREFETCH
  // Loads run ahead of the round that uses them (other slots: no ordering with this round's
  // stores), so the round loop is not a chain of dependent load latencies: stage bytes two rounds
  // ahead, a finished path's pixel and radiance one round ahead (issued once its stage byte, loaded
  // the round before, is known).
  int stage_n1 = P.stage[r0 + lane];
  int stage_n2 = r0 + 32 < r1 ? P.stage[r0 + 32 + lane] : 0;
  int pix_n1 = 0;
  v3 L_n1 = mk3(0.0, 0.0, 0.0);
  if (LW_GEN_PREFETCH > 1 && regen && stage_n1 == LW_STAGE_TERMINATED) {
    pix_n1 = P.pix[r0 + lane];
    L_n1 = load_L(P, r0 + lane, CMP);
  }
#endif
  for (int base = r0; base < r1; base += 32) {
    int s = base + lane;
#if LW_GEN_PREFETCH
    const int stage0 = stage_n1;
    const int fpix = pix_n1;
    const v3 fL = L_n1;
    stage_n1 = stage_n2;
    if (base + 64 < r1) stage_n2 = P.stage[s + 64];
    if (LW_GEN_PREFETCH > 1 && regen && base + 32 < r1 && stage_n1 == LW_STAGE_TERMINATED) {
      pix_n1 = P.pix[s + 32];
      L_n1 = load_L(P, s + 32, CMP);
    }
    int stage = stage0;
#else
    int stage = P.stage[s];
#endif
    bool flushed = false;
    if (regen && stage == LW_STAGE_TERMINATED) {
#if LW_GEN_PREFETCH > 1
      bad += lw_accumulate(fb, fpix, fL);
#else
      bad += lw_accumulate(fb, P.pix[s], load_L(P, s, CMP));
#endif
      paths++;
      stage = LW_STAGE_GENERATE;
      flushed = true;
    }
    bool want = regen && stage == LW_STAGE_GENERATE;
    bool trace = stage == LW_STAGE_TRACE;
    unsigned mw = __ballot_sync(0xffffffffu, want), mt = __ballot_sync(0xffffffffu, trace);
    if (!(mw | mt)) continue;
    int pw = __popc(mw & lt), pt = __popc(mt & lt);
    int avail = min(gleft, __popc(mw));
    if (want) {
      if (pw < avail) {
        long long item = wnext + pw;
        int pix;
        long long index = work_index(S, w, item, pix);
        PathState ps;
        lw_path_init<CMP>(S, index, ps);
        store_state(P, s, ps, needs_nprev(S), CMP);
        if (LPE) P.lpe_state[s] = lw_lpe_step(&lpe, lpe.start, LW_EV_C);
        P.pix[s] = pix;
        P.stage[s] = LW_STAGE_TRACE;
        trace = true;
      } else if (flushed) {
        P.stage[s] = LW_STAGE_GENERATE;
      }
    }
    if (trace) P.q_ext[enext + pt + min(pw, avail)] = s;
    wnext += avail;
    gleft -= avail;
    enext += __popc(mt) + avail;
  }
  warp_add(&cnt->nonfinite, bad);
  warp_add(&cnt->paths, paths);
}

template <bool COUNT, int NODES, bool CMP>
__global__ void __launch_bounds__(128, LW_TRACE_MINB) k_trace_ext(DevScene S, Pool P, Counters* __restrict__ cnt, int nrnodes, int use_smem) {
  extern __shared__ __align__(16) unsigned char smem[];
  RenderBVH bvh = stage_bvh(S.bvh, nrnodes, smem, use_smem != 0);
  int n = cnt->n_ext;
  const bool tail = cnt->tail != 0;
  LwTraceCount tc;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    int k = base + threadIdx.x;
    if (k < n) {
      int s = P.q_ext[k];
      if (tail && P.stage[s] != LW_STAGE_TRACE) continue;  // finished entry of the tail queue
      double o[3], d[3];
      load_ray(P, s, o, d, CMP);
      LwHit h;
      lw_trace_closest<COUNT, NODES, (LW_SPEC_SMEM & 1) != 0>(bvh, o, d, INFINITY, h, &tc);
      P.hit0[s] = make_double2(h.t, h.bu);
      P.hit1[s] = make_double2(h.bv, __longlong_as_double(h.tri));
    }
  }
  if (COUNT) {
    warp_add(&cnt->ext_nodes, tc.nodes);
    warp_add(&cnt->ext_tris, tc.tris);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cnt->rays_ext += (unsigned long long)(cnt->tail ? cnt->n_trace : n);
    cnt->waves += 1;
  }
}


// Persistent extension trace over a global-memory BVH with lane refill (Aila & Laine 2009): a lane
// whose ray is finished takes the next queue entry (one warp-aggregated atomic per refill) instead
// of idling until the slowest lane of its warp is done, so the warp's SIMT efficiency does not
// collapse on incoherent rays.  The traversal is the same as lw_trace_closest (same visit order,
// same hits); the loop yields after every leaf so that refills can happen.
template <bool COUNT, int NODES, bool CMP>
__global__ void __launch_bounds__(128, LW_TRACE_MINB) k_trace_ext_p(DevScene S, Pool P, Counters* __restrict__ cnt,
                                                                    int nrnodes) {
  extern __shared__ __align__(16) unsigned char smem[];
  RenderBVH bvh = stage_bvh(S.bvh, nrnodes, smem, NODES == LW_NODES_SMEM);
  const int n = cnt->n_ext;
  const bool tail = cnt->tail != 0;
  const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
  LwTraceCount tc;
  int s = -1;
  LwRayF r;
  double ht = 0.0, hu = 0.0, hv = 0.0, best_det = 1.0;
  long long htri = -1;
  float best = 0.0f;
  int ref = LW_REF_NONE, sp = 0;
  unsigned long long stk[LW_STACK];
  bool more = true;
  for (;;) {
    unsigned idle = __ballot_sync(0xffffffffu, s < 0);
    if (more && __popc(idle) >= (idle == 0xffffffffu ? 1 : LW_REFILL)) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&cnt->ext_next, __popc(idle));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + __popc(idle) >= n) more = false;
      if (s < 0) {
        int k = base + __popc(idle & lt);
        if (k < n && (!tail || P.stage[P.q_ext[k]] == LW_STAGE_TRACE)) {
          s = P.q_ext[k];
          double o[3], d[3];
          load_ray(P, s, o, d, CMP);
          lw_rayf_setup(r, bvh, o, d);
          ht = INFINITY;
          hu = hv = 0.0;
          best_det = 1.0;
          htri = -1;
          best = INFINITY;
          sp = 0;
          ref = bvh.ntris == 0 ? LW_REF_NONE : bvh.root_ref;
        }
      }
    }
    if (__all_sync(0xffffffffu, s < 0) && !more) break;  // (tail queue: a refill may hit only finished entries)
    if (s < 0) continue;
#if LW_SPEC & 1
    // speculative traversal (Aila & Laine 2009): a lane that reaches a leaf postpones it and keeps
    // descending until every lane of the warp holds a leaf, so the node loop and the leaf loop
    // each run with more lanes active.  Visit order changes, the closest hit does not.
    int leaf = LW_REF_NONE;
    if (ref < 0) {
      leaf = ref;
      ref = lw_pop_cull(stk, sp, best);
    }
    while (ref >= 0 && ref != LW_REF_NONE) {
      float tn[4];
      int cr[4];
      unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
      if (COUNT) tc.nodes++;
      int nh = __popc(m);
      if (nh <= 1) {
        ref = nh == 0 ? lw_pop_cull(stk, sp, best) : lw_pick(m, cr);
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++)
          if (!(m & (1u << c))) tn[c] = INFINITY;
        lw_cswap(tn[0], cr[0], tn[1], cr[1]);
        lw_cswap(tn[2], cr[2], tn[3], cr[3]);
        lw_cswap(tn[0], cr[0], tn[2], cr[2]);
        lw_cswap(tn[1], cr[1], tn[3], cr[3]);
        lw_cswap(tn[1], cr[1], tn[2], cr[2]);
        if (nh > 3) stk[sp++] = lw_stk_pack(cr[3], tn[3]);
        if (nh > 2) stk[sp++] = lw_stk_pack(cr[2], tn[2]);
        stk[sp++] = lw_stk_pack(cr[1], tn[1]);
        ref = cr[0];
      }
      if (ref < 0 && leaf == LW_REF_NONE) {
        leaf = ref;
        ref = lw_pop_cull(stk, sp, best);
      }
      if (!__any_sync(__activemask(), leaf == LW_REF_NONE)) break;
    }
    if (leaf == LW_REF_NONE && ref < 0) {
      leaf = ref;
      ref = lw_pop_cull(stk, sp, best);
    }
    if (leaf != LW_REF_NONE) {
      int v = -leaf - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) tc.tris++;
        double t, bu, bv, det;
        if (!lw_tri_eval(bvh.tris[k].v, r.sh, t, bu, bv, det) || t <= 0.0 || t > ht) continue;
        long long id = bvh.tris[k].id;
        if (t == ht && htri >= 0 && id >= htri) continue;
        ht = t;
        htri = id;
        hu = bu;
        hv = bv;
        best_det = det;
        best = __double2float_ru(t);
      }
    }
    if (ref == LW_REF_NONE) {
      P.hit0[s] = make_double2(ht, htri >= 0 ? hu / best_det : 0.0);
      P.hit1[s] = make_double2(htri >= 0 ? hv / best_det : 0.0, __longlong_as_double(htri));
      s = -1;
    }
  }
#else
    // descend to the next leaf
    while (ref >= 0 && ref != LW_REF_NONE) {
      float tn[4];
      int cr[4];
      unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
      if (COUNT) tc.nodes++;
      int nh = __popc(m);
      if (nh <= 1) {
        ref = nh == 0 ? LW_REF_NONE : lw_pick(m, cr);
        if (nh == 0) break;
        continue;
      }
#pragma unroll
      for (int c = 0; c < 4; c++)
        if (!(m & (1u << c))) tn[c] = INFINITY;
      lw_cswap(tn[0], cr[0], tn[1], cr[1]);
      lw_cswap(tn[2], cr[2], tn[3], cr[3]);
      lw_cswap(tn[0], cr[0], tn[2], cr[2]);
      lw_cswap(tn[1], cr[1], tn[3], cr[3]);
      lw_cswap(tn[1], cr[1], tn[2], cr[2]);
      if (nh > 3) stk[sp++] = lw_stk_pack(cr[3], tn[3]);
      if (nh > 2) stk[sp++] = lw_stk_pack(cr[2], tn[2]);
      stk[sp++] = lw_stk_pack(cr[1], tn[1]);
      ref = cr[0];
    }
    if (ref != LW_REF_NONE) {
      int v = -ref - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) tc.tris++;
        double t, bu, bv, det;
        if (!lw_tri_eval(bvh.tris[k].v, r.sh, t, bu, bv, det) || t <= 0.0 || t > ht) continue;
        long long id = bvh.tris[k].id;
        if (t == ht && htri >= 0 && id >= htri) continue;
        ht = t;
        htri = id;
        hu = bu;
        hv = bv;
        best_det = det;
        best = __double2float_ru(t);
      }
    }
    ref = LW_REF_NONE;
    while (sp > 0) {
      unsigned long long e = stk[--sp];
      if (__uint_as_float((unsigned)(e >> 32)) <= best) {
        ref = (int)(unsigned)e;
        break;
      }
    }
    if (ref == LW_REF_NONE) {
      P.hit0[s] = make_double2(ht, htri >= 0 ? hu / best_det : 0.0);
      P.hit1[s] = make_double2(htri >= 0 ? hv / best_det : 0.0, __longlong_as_double(htri));
      s = -1;
    }
  }
#endif
  if (COUNT) {
    warp_add(&cnt->ext_nodes, tc.nodes);
    warp_add(&cnt->ext_tris, tc.tris);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cnt->rays_ext += (unsigned long long)(cnt->tail ? cnt->n_trace : n);
    cnt->waves += 1;
  }
}

__device__ __forceinline__ void load_hit(const Pool& P, int s, LwHit& h) {
  double2 h0 = P.hit0[s], h1 = P.hit1[s];
  h.t = h0.x;
  h.bu = h0.y;
  h.bv = h1.x;
  h.tri = __double_as_longlong(h1.y);
}

// NEE half of the material stage (runs before k_shade so it sees the incoming throughput):
// light / environment sample, BSDF evaluation, shadow-ray setup
template <bool LPE, bool LT, bool CMP, int MC>
__global__ void __launch_bounds__(128, (MC & LW_MC_DIFFUSE) ? LW_NEE_MINB_D : LW_NEE_MINB) k_shade_nee(DevScene S, Pool P, Counters* __restrict__ cnt,
                                                                LwLpe lpe) {
  extern __shared__ __align__(16) unsigned char smem[];
  LwLightTree lt;
  if (LT) lt = lw_lt_stage(S.lt, S.lt_nheap, smem);
  int n = cnt->n_ext;
  const bool tail = cnt->tail != 0;
  const int stride = gridDim.x * blockDim.x;
  // LW_SHADE_PREFETCH 1: queue entries read one grid stride ahead; 2: two strides ahead, and the
  // next entry's hit record and flags one stride ahead
  const int k0 = blockIdx.x * blockDim.x + threadIdx.x;
  int s_next = LW_SHADE_PREFETCH && k0 < n ? P.q_ext[k0] : 0;
  int s_next2 = LW_SHADE_PREFETCH > 1 && k0 + stride < n ? P.q_ext[k0 + stride] : 0;
  double2 h0n = make_double2(0.0, 0.0), h1n = make_double2(0.0, 0.0);
  int fn = 0;
  if (LW_SHADE_PREFETCH > 1 && k0 < n) {
    h0n = P.hit0[s_next];
    h1n = P.hit1[s_next];
    fn = P.flags[s_next];
  }
  for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
    int k = base + threadIdx.x;
    bool valid = k < n;
    int s = 0;
    bool shadow = false;
    const int s_cur = s_next;
    const double2 h0c = h0n, h1c = h1n;
    const int fc = fn;
    if (LW_SHADE_PREFETCH > 1) {
      s_next = s_next2;
      if (k + 2 * stride < n) s_next2 = P.q_ext[k + 2 * stride];
      if (k + stride < n) {
        h0n = P.hit0[s_next];
        h1n = P.hit1[s_next];
        fn = P.flags[s_next];
      }
    } else if (LW_SHADE_PREFETCH && k + stride < n) {
      s_next = P.q_ext[k + stride];
    }
    if (valid) {
      s = LW_SHADE_PREFETCH ? s_cur : P.q_ext[k];
      LwHit h;
      int f;
      if (LW_SHADE_PREFETCH > 1) {
        h.t = h0c.x;
        h.bu = h0c.y;
        h.bv = h1c.x;
        h.tri = __double_as_longlong(h1c.y);
        f = fc;
      } else {
        load_hit(P, s, h);
        f = P.flags[s];
      }
      int bounce = f & F_BOUNCE;
      if (h.tri >= 0 && bounce != S.max_depth - 1 && (!tail || P.stage[s] == LW_STAGE_TRACE)) {
        PathState ps;
        if (CMP) {
          ps.d = lw_oct_dir((unsigned)((unsigned long long)__double_as_longlong(P.ray1[s].y) >> 32));
          float4 t0 = reinterpret_cast<const float4*>(P.tp0)[s];
          ps.beta = mk3((double)t0.x, (double)t0.y, (double)t0.z);
          ps.index = __double_as_longlong(P.tp1[s].y);
        } else {
          double2 a = P.ray1[s], c = P.ray2[s];
          ps.d = mk3(a.y, c.x, c.y);
          double2 t0 = P.tp0[s], t1 = P.tp1[s];
          ps.beta = mk3(t0.x, t0.y, t1.x);
          ps.index = __double_as_longlong(P.misc[s].y);
        }
        ps.bounce = bounce;
        if (LPE) ps.lpe = P.lpe_state[s];
        ShadeGeom g;
        double w;
        lw_shade_hit(S, ps.d, h, g, w);
        lw_shade_frame<MC>(S, ps.d, h, w, g);
        ShadowRay sh;
        lw_shade_nee<MC>(S, ps, g, sh, LPE ? &lpe : nullptr, LT ? &lt : nullptr);
        shadow = sh.valid != 0;
        if (LPE && shadow) {
          P.sh5[s] = make_double2(sh.c_diffuse.x, sh.c_diffuse.y);
          P.sh6[s] = make_double2(sh.c_diffuse.z, sh.c_glossy.x);
          P.sh7[s] = make_double2(sh.c_glossy.y, sh.c_glossy.z);
          P.sh_lpe[s] = sh.lpe | (sh.term << 16);
        }
        if (shadow) {
          P.sh0[s] = make_double2(sh.o.x, sh.o.y);
          P.sh1[s] = make_double2(sh.o.z, sh.d.x);
          P.sh2[s] = make_double2(sh.d.y, sh.d.z);
          P.sh3[s] = make_double2(sh.tmax, sh.contrib.x);
          P.sh4[s] = make_double2(sh.contrib.y, sh.contrib.z);
        }
      }
    }
    int q = warp_push(&cnt->n_shadow, valid && shadow);
    if (q >= 0) P.q_shadow[q] = s;
  }
}

// material half: miss/emission (MIS), BSDF sampling, Russian roulette, next ray, stage tag
template <bool LPE, bool LT, bool CMP, int MC>
__global__ void __launch_bounds__(128, (MC & LW_MC_DIFFUSE) ? LW_SHADE_MINB_D : LW_SHADE_MINB) k_shade(DevScene S, Pool P, Counters* __restrict__ cnt, LwLpe lpe) {
  extern __shared__ __align__(16) unsigned char smem[];
  LwLightTree lt;
  if (LT) lt = lw_lt_stage(S.lt, S.lt_nheap, smem);
  int n = cnt->n_ext;
  const bool tail = cnt->tail != 0;
  unsigned long long alive_count = 0;
  const int stride = gridDim.x * blockDim.x;
  // queue entries read one grid stride ahead (the general-material kernel spills more with the
  // extra live value: C4 k_shade +4 %, so it keeps the plain load)
  constexpr bool PF = LW_SHADE_PREFETCH && (MC & LW_MC_DIFFUSE);
  constexpr bool PF2 = PF && LW_SHADE_K2;  // two-deep: the next entry's hit record one stride ahead
  const int k0 = blockIdx.x * blockDim.x + threadIdx.x;
  int s_next = PF && k0 < n ? P.q_ext[k0] : 0;
  int s_next2 = PF2 && k0 + stride < n ? P.q_ext[k0 + stride] : 0;
  double2 h0n = make_double2(0.0, 0.0), h1n = make_double2(0.0, 0.0);
  if (PF2 && k0 < n) {
    h0n = P.hit0[s_next];
    h1n = P.hit1[s_next];
  }
  for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
    int k = base + threadIdx.x;
    const int s_cur = s_next;
    const double2 h0c = h0n, h1c = h1n;
    if (PF2) {
      s_next = s_next2;
      if (k + 2 * stride < n) s_next2 = P.q_ext[k + 2 * stride];
      if (k + stride < n) {
        h0n = P.hit0[s_next];
        h1n = P.hit1[s_next];
      }
    } else if (PF && k + stride < n) {
      s_next = P.q_ext[k + stride];
    }
    if (k < n) {
      int s = PF ? s_cur : P.q_ext[k];
      if (tail && P.stage[s] != LW_STAGE_TRACE) continue;  // finished entry of the tail queue
      PathState ps;
      load_state(P, s, ps, needs_nprev<MC>(S), CMP);
      LwHit h;
      if (PF2) {
        h.t = h0c.x;
        h.bu = h0c.y;
        h.bv = h1c.x;
        h.tri = __double_as_longlong(h1c.y);
      } else {
        load_hit(P, s, h);
      }
      ShadeGeom g;
      double w;
      bool alive = false;
      if (LPE) ps.lpe = P.lpe_state[s];
      if (lw_shade_emission<CMP, MC>(S, ps, h, g, w, LPE ? &lpe : nullptr, LPE ? P.pix[s] : 0, LT ? &lt : nullptr)) {
        lw_shade_frame<MC>(S, ps.d, h, w, g);
        alive = lw_shade_material<CMP, MC>(S, ps, g, LPE ? &lpe : nullptr);
      }
      store_state(P, s, ps, needs_nprev<MC>(S), CMP);
      if (LPE) P.lpe_state[s] = ps.lpe;
      P.stage[s] = alive ? LW_STAGE_TRACE : LW_STAGE_TERMINATED;
      alive_count += alive ? 1 : 0;
    }
  }
  warp_add(&cnt->n_alive_ull, alive_count);
}

// an unoccluded shadow ray adds its NEE contribution (and routes its LPE split)
template <bool LPE, bool compact>
__device__ __forceinline__ void shadow_unoccluded(const Pool& P, int s, double cx, const LwLpe& lpe) {
  double2 f = P.sh4[s];
  if (compact) {  // L = q32(L + contribution), as lw_q32v in the megakernel and the oracle
    float4* t0p = reinterpret_cast<float4*>(P.tp0) + s;
    float4 t0 = *t0p;
    double2 t1 = P.tp1[s];
    unsigned long long lb = (unsigned long long)__double_as_longlong(t1.x);
    t0.w = __double2float_rn((double)t0.w + cx);
    double ly = lw_q32((double)__uint_as_float((unsigned)lb) + f.x);
    double lz = lw_q32((double)__uint_as_float((unsigned)(lb >> 32)) + f.y);
    *t0p = t0;
    t1.x = __longlong_as_double((long long)pack2f(ly, lz));
    P.tp1[s] = t1;
  } else {
    double2 t1 = P.tp1[s], t2 = P.tp2[s];
    t1.y = t1.y + cx;
    t2.x = t2.x + f.x;
    t2.y = t2.y + f.y;
    P.tp1[s] = t1;
    P.tp2[s] = t2;
  }
  if (LPE) {
    double2 a5 = P.sh5[s], a6 = P.sh6[s], a7 = P.sh7[s];
    int sl = P.sh_lpe[s], st0 = sl & 0xffff, term = sl >> 16;
    long long pix = P.pix[s];
    lw_lpe_route(&lpe, lw_lpe_step(&lpe, lw_lpe_step(&lpe, st0, LW_EV_RD), term), pix, mk3(a5.x, a5.y, a6.x));
    lw_lpe_route(&lpe, lw_lpe_step(&lpe, lw_lpe_step(&lpe, st0, LW_EV_RG), term), pix, mk3(a6.y, a7.x, a7.y));
  }
}

// persistent any-hit trace over a global-memory BVH with lane refill (see k_trace_ext_p)
template <bool COUNT, bool LPE, int NODES, bool CMP>
__global__ void __launch_bounds__(128, LW_SHADOW_MINB) k_trace_shadow_p(DevScene S, Pool P, Counters* __restrict__ cnt,
                                                                        int nrnodes, LwLpe lpe) {
  extern __shared__ __align__(16) unsigned char smem[];
  RenderBVH bvh = stage_bvh(S.bvh, nrnodes, smem, NODES == LW_NODES_SMEM);
  const int n = cnt->n_shadow;
  const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
  LwTraceCount tc;
  int s = -1;
  LwRayF r;
  double tmax = 0.0, cx = 0.0;
  float best = 0.0f;
  int ref = LW_REF_NONE, sp = 0;
  int stk[LW_STACK];
  bool more = true;
  for (;;) {
    unsigned idle = __ballot_sync(0xffffffffu, s < 0);
    if (more && __popc(idle) >= (idle == 0xffffffffu ? 1 : LW_REFILL)) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&cnt->sh_next, __popc(idle));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + __popc(idle) >= n) more = false;
      if (s < 0) {
        int k = base + __popc(idle & lt);
        if (k < n) {
          s = P.q_shadow[k];
          double2 a = P.sh0[s], b = P.sh1[s], c = P.sh2[s], e = P.sh3[s];
          double o[3] = {a.x, a.y, b.x}, d[3] = {b.y, c.x, c.y};
          lw_rayf_setup(r, bvh, o, d);
          tmax = e.x;
          cx = e.y;
          best = __double2float_ru(tmax);
          sp = 0;
          ref = bvh.ntris == 0 ? LW_REF_NONE : bvh.root_ref;
        }
      }
    }
    if (__all_sync(0xffffffffu, s < 0)) break;
    if (s < 0) continue;
    bool occluded = false;
#if LW_SPEC & 2
    int leaf = LW_REF_NONE;
    if (ref < 0) {
      leaf = ref;
      ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
    }
    while (ref >= 0 && ref != LW_REF_NONE) {
      float tn[4];
      int cr[4];
      unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
      if (COUNT) tc.nodes++;
      if (m == 0) {
        ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
      } else {
        ref = lw_pick(m, cr);
        m &= m - 1;
#pragma unroll
        for (int c = 1; c < 4; c++)
          if (m & (1u << c)) stk[sp++] = cr[c];
      }
      if (ref < 0 && leaf == LW_REF_NONE) {
        leaf = ref;
        ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
      }
      if (!__any_sync(__activemask(), leaf == LW_REF_NONE)) break;
    }
    if (leaf == LW_REF_NONE && ref < 0) {
      leaf = ref;
      ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
    }
    if (leaf != LW_REF_NONE) {
      int v = -leaf - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) tc.tris++;
        if (lw_tri_occludes(bvh.tris[k].v, r.sh, tmax)) {
          occluded = true;
          break;
        }
      }
    }
    if (occluded || ref == LW_REF_NONE) {
      if (!occluded) {
        shadow_unoccluded<LPE, CMP>(P, s, cx, lpe);
        if (COUNT) tc.lit++;
      }
      s = -1;
    }
  }
#else
    while (ref >= 0 && ref != LW_REF_NONE) {
      float tn[4];
      int cr[4];
      unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
      if (COUNT) tc.nodes++;
      if (m == 0) {
        ref = LW_REF_NONE;
        break;
      }
      ref = lw_pick(m, cr);
      m &= m - 1;
#pragma unroll
      for (int c = 1; c < 4; c++)
        if (m & (1u << c)) stk[sp++] = cr[c];
    }
    if (ref != LW_REF_NONE) {
      int v = -ref - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) tc.tris++;
        if (lw_tri_occludes(bvh.tris[k].v, r.sh, tmax)) {
          occluded = true;
          break;
        }
      }
    }
    ref = sp > 0 && !occluded ? stk[--sp] : LW_REF_NONE;
    if (ref == LW_REF_NONE) {
      if (!occluded) {
        shadow_unoccluded<LPE, CMP>(P, s, cx, lpe);
        if (COUNT) tc.lit++;
      }
      s = -1;
    }
  }
#endif
  if (COUNT) {
    warp_add(&cnt->sh_nodes, tc.nodes);
    warp_add(&cnt->sh_tris, tc.tris);
    warp_add(&cnt->sh_unocc, tc.lit);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt->rays_shadow += (unsigned long long)n;
}

template <bool COUNT, bool LPE, int NODES, bool CMP>
__global__ void __launch_bounds__(128, LW_SHADOW_MINB) k_trace_shadow(DevScene S, Pool P, Counters* __restrict__ cnt, int nrnodes, int use_smem,
                                                                      LwLpe lpe) {
  extern __shared__ __align__(16) unsigned char smem[];
  RenderBVH bvh = stage_bvh(S.bvh, nrnodes, smem, use_smem != 0);
  int n = cnt->n_shadow;
  LwTraceCount tc;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    int k = base + threadIdx.x;
    if (k < n) {
      int s = P.q_shadow[k];
      double2 a = P.sh0[s], b = P.sh1[s], c = P.sh2[s], e = P.sh3[s];
      double o[3] = {a.x, a.y, b.x}, d[3] = {b.y, c.x, c.y};
      if (!lw_trace_any<COUNT, NODES, (LW_SPEC_SMEM & 2) != 0>(bvh, o, d, e.x, &tc)) {
        shadow_unoccluded<LPE, CMP>(P, s, e.y, lpe);
        if (COUNT) tc.lit++;
      }
    }
  }
  if (COUNT) {
    warp_add(&cnt->sh_nodes, tc.nodes);
    warp_add(&cnt->sh_tris, tc.tris);
    warp_add(&cnt->sh_unocc, tc.lit);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt->rays_shadow += (unsigned long long)n;
}

// n_alive is accumulated as 64-bit by k_shade; fold it into the 32-bit field the decision reads
__global__ void k_wave_end(Counters* cnt) {
  cnt->n_alive = (int)cnt->n_alive_ull;
  cnt->n_alive_ull = 0;
}

// megakernel tail: run every in-flight path to completion, in pool order
template <bool LPE, bool CMP>
__global__ void __launch_bounds__(128) k_mega_tail(DevScene S, Pool P, unsigned long long* __restrict__ fb,
                                                   Counters* __restrict__ cnt, int nrnodes, int use_smem, LwLpe lpe) {
  extern __shared__ __align__(16) unsigned char smem[];
  RenderBVH bvh = stage_bvh(S.bvh, nrnodes, smem, use_smem != 0);
  unsigned long long next = 0, nsh = 0, bad = 0, paths = 0;
  for (int base = blockIdx.x * blockDim.x; base < P.size; base += gridDim.x * blockDim.x) {
    int s = base + threadIdx.x;
    if (s < P.size && P.stage[s] == LW_STAGE_TRACE) {
      PathState ps;
      load_state(P, s, ps, needs_nprev(S), CMP);
      if (LPE) ps.lpe = P.lpe_state[s];
      run_to_completion<CMP>(S, bvh, ps, next, nsh, LPE ? &lpe : nullptr, P.pix[s]);
      bad += lw_accumulate(fb, P.pix[s], ps.L);
      paths++;
      P.stage[s] = LW_STAGE_GENERATE;
    }
  }
  warp_add(&cnt->rays_ext, next);
  warp_add(&cnt->rays_shadow, nsh);
  warp_add(&cnt->nonfinite, bad);
  warp_add(&cnt->paths, paths);
}

__global__ void k_tail_done(Counters* cnt) { cnt->n_alive = 0; }

// LW_INSTR_TIME: %globaltimer (ns) and the stage starting now, appended to the pass's stamp list;
// consecutive stamps bracket one stage (works inside CUDA graphs, unlike event records)
__global__ void k_stamp(unsigned long long* stamps, Counters* cnt, int stage, int cap) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  int i = cnt->stamp_n;
  if (i < cap) {
    stamps[i] = (t << 4) | (unsigned long long)stage;
    cnt->stamp_n = i + 1;
  }
}

// end of a wave inside the CUDA-graph loop: run another while work is left or paths are alive
__global__ void k_wave_cond(Counters* cnt, cudaGraphConditionalHandle h, int max_waves) {
  const long long total = cnt->wr.nits * cnt->wr.npix;
  int gw = ++cnt->gwaves;
  bool more = (long long)cnt->work_next < total || cnt->n_alive > 0;
  if (more && gw >= max_waves) {
    cnt->overflow = 1;
    more = false;
  }
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

// pass totals into the context's running statistics (device-side, so passes can queue up)
__global__ void k_stats_accum(const Counters* cnt, unsigned long long* acc) {
  acc[0] += cnt->paths;
  acc[1] += cnt->rays_ext;
  acc[2] += cnt->rays_shadow;
  acc[3] += cnt->nonfinite;
  acc[4] += cnt->waves;
  acc[5] += cnt->regens;
}

// ---- debug / parity kernels -------------------------------------------------------------

__global__ void k_trace_closest_dbg(DevScene S, const double* o, const double* d, const double* tm, long long n,
                                    double* ot, long long* otri, double* ob) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  LwHit h;
  lw_trace_closest(S.bvh, oo, dd, tm[i], h);
  bool hit = h.tri >= 0;
  ot[i] = hit ? h.t : 1e308;
  otri[i] = hit ? h.tri : -1;
  ob[2 * i] = hit ? h.bu : 0.0;
  ob[2 * i + 1] = hit ? h.bv : 0.0;
}

// ---- known-answer surface of the render math ----------------
// BSDF evaluate / sample in the local shading frame (z = shading normal), layer weights from wo.z
__global__ void k_bsdf_eval_dbg(lw_material m, const double* wo, const double* wi, long long n, double* of,
                                double* op) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v3 a = lw_ld3(wo + 3 * i), b = lw_ld3(wi + 3 * i);
  LayerW lw;
  lw_layer_weights(m, a.z, lw);
  double pdf;
  v3 f = lw_bsdf_eval(m, lw, a, b, pdf);
  of[3 * i] = f.x;
  of[3 * i + 1] = f.y;
  of[3 * i + 2] = f.z;
  op[i] = pdf;
}

__global__ void k_bsdf_sample_dbg(lw_material m, const double* wo, const int* front, const double* uv, long long n,
                                  double* owi, double* ow, double* op, int* oflags) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v3 a = lw_ld3(wo + 3 * i);
  LayerW lw;
  lw_layer_weights(m, a.z, lw);
  BSample bs;
  bs.wi = bs.weight = mk3(0.0, 0.0, 0.0);
  bs.pdf = 0.0;
  bs.delta = bs.transmit = bs.event = 0;
  bool ok = lw_bsdf_sample(m, lw, a, front[i] != 0, uv[2 * i], uv[2 * i + 1], bs);
  owi[3 * i] = bs.wi.x;
  owi[3 * i + 1] = bs.wi.y;
  owi[3 * i + 2] = bs.wi.z;
  ow[3 * i] = bs.weight.x;
  ow[3 * i + 1] = bs.weight.y;
  ow[3 * i + 2] = bs.weight.z;
  op[i] = bs.pdf;
  oflags[i] = (ok ? 1 : 0) | (bs.delta ? 2 : 0) | (bs.transmit ? 4 : 0) | (bs.event << 8);
}

__global__ void k_mis_dbg(const double* a, const double* b, long long n, double* o) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) o[i] = lw_mis_balance(a[i], b[i]);
}

__global__ void k_nee_light_dbg(DevScene S, const double* p, const double* ngf, const double* uv, long long n,
                                double* owi, double* oLe, double* opdf, double* otmax, long long* oe) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v3 wi, Le;
  double pl, tm;
  long long e;
  bool ok = lw_nee_light_sample(S, lw_ld3(p + 3 * i), lw_ld3(ngf + 3 * i), uv[2 * i], uv[2 * i + 1], nullptr, wi, Le,
                                pl, tm, e);
  owi[3 * i] = wi.x;
  owi[3 * i + 1] = wi.y;
  owi[3 * i + 2] = wi.z;
  oLe[3 * i] = Le.x;
  oLe[3 * i + 1] = Le.y;
  oLe[3 * i + 2] = Le.z;
  opdf[i] = ok ? pl : 0.0;
  otmax[i] = tm;
  oe[i] = e;
}

// what BSDF sampling sees along (o, d): emitted radiance and the light-sampling pdf MIS weighs it
// against (emitter hit: lw_emitter_hit_pdf; miss: the environment's lw_env_eval); e = emitter,
// -1 environment, -2 a non-emissive surface (pdf 0)
__global__ void k_emission_pdf_dbg(DevScene S, const double* o, const double* d, const int* nprev, long long n,
                                   double* oLe, double* opdf, long long* oe) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  LwHit h;
  lw_trace_closest(S.bvh, oo, dd, INFINITY, h);
  v3 dv = mk3(dd[0], dd[1], dd[2]);
  v3 Le = mk3(0.0, 0.0, 0.0);
  double pdf = 0.0;
  long long e = -2;
  if (h.tri < 0) {
    e = -1;
    Le = lw_env_eval(S, dv, nprev[i], pdf);
  } else {
    ShadeGeom g;
    double w;
    lw_shade_hit(S, dv, h, g, w);
    int k = S.emit_of_tri[h.tri];
    if (k >= 0 && S.nemit > 0 && (g.front || S.emit_two[k])) {
      e = k;
      Le = lw_ld3(S.emit_rad + 3 * k);
      pdf = lw_emitter_hit_pdf(S, k, mk3(oo[0], oo[1], oo[2]), nprev[i], g.ng, dv, h.t, nullptr);
    }
  }
  oLe[3 * i] = Le.x;
  oLe[3 * i + 1] = Le.y;
  oLe[3 * i + 2] = Le.z;
  opdf[i] = pdf;
  oe[i] = e;
}

__global__ void k_trace_any_dbg(DevScene S, const double* o, const double* d, const double* tm, long long n, int* occ) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  occ[i] = lw_trace_any(S.bvh, oo, dd, tm[i]) ? 1 : 0;
}

__global__ void k_camera_dbg(DevScene S, const long long* idx, long long n, double* oo, double* od) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v3 o, d;
  lw_camera_ray(S, idx[i], o, d);
  oo[3 * i] = o.x;
  oo[3 * i + 1] = o.y;
  oo[3 * i + 2] = o.z;
  od[3 * i] = d.x;
  od[3 * i + 1] = d.y;
  od[3 * i + 2] = d.z;
}

__global__ void k_light_sample_dbg(DevScene S, const double* x, const double* nrm, const double* u, long long n,
                                   long long* oe, double* op, double* ou) {
  extern __shared__ __align__(16) unsigned char smem[];
  LwLightTree T = lw_lt_stage(S.lt, S.lt_nheap, smem);
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ps, uo;
  oe[i] = lw_lt_sample(T, lw_ld3(x + 3 * i), lw_ld3(nrm + 3 * i), u[i], ps, uo);
  op[i] = ps;
  ou[i] = uo;
}

__global__ void k_light_pdf_dbg(DevScene S, const long long* e, const double* x, const double* nrm, long long n,
                                double* op) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  op[i] = lw_lt_pdf(S.lt, e[i], lw_ld3(x + 3 * i), lw_ld3(nrm + 3 * i));  // global nodes only
}

__global__ void k_env_sample_dbg(DevScene S, const long long* pk, const double* uv, long long n, long long* ot,
                                 double* op, double* ouv) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long row, col;
  double p, u, v;
  lw_ep_sample(S.env_pyr, lw_ep_bin(pk[i]), uv[2 * i], uv[2 * i + 1], row, col, p, u, v);
  ot[i] = row * S.env_w + col;
  op[i] = p;
  ouv[2 * i] = u;
  ouv[2 * i + 1] = v;
}

__global__ void k_env_pdf_dbg(DevScene S, const long long* pk, const long long* tx, long long n, double* op) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  op[i] = lw_ep_pdf(S.env_pyr, lw_ep_bin(pk[i]), tx[i] / S.env_w, tx[i] % S.env_w);
}

__global__ void k_resolve(const unsigned long long* fb, long long n, double scale, float* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)((double)(long long)fb[i] * scale);
}

// dynamic shared memory of the light-hierarchy top (0 without a hierarchy)
size_t lt_smem_bytes(const lw_ctx* c) {
  if (c->S.light_mode != LW_LIGHTS_TREE) return 0;
  return sizeof(LwLightNode) * (size_t)std::min(c->S.lt_nheap, LW_LT_SMEM_NODES);
}

int nrnodes_of(const lw_ctx* c) { return c->ref_bvh.nnodes > 1 ? (int)((c->ref_bvh.nnodes - 1) / 2) : 0; }

// binary tree -> 4-wide nodes, one launch per binary level (frontier in device memory)
int collapse_wide(lw_ctx* c, const SahNode* bn, int nr, int root_ref, int levels, WNode* out, int& max_need) {
  max_need = 0;
  if (nr <= 0 || root_ref < 0) return LW_OK;
  cudaStream_t st = c->stream;
  DevBuf f0, f1, need, cnt;
  // stream-ordered scratch like the rest of the upload (a synchronous cudaMalloc here stalled on
  // the reserved pool memory: 2 -> 386 ms over five C3 uploads)
  LW_CUDA_TRY(f0.alloc(sizeof(int) * nr, st));
  LW_CUDA_TRY(f1.alloc(sizeof(int) * nr, st));
  LW_CUDA_TRY(need.alloc(sizeof(int) * nr, st));
  LW_CUDA_TRY(cnt.alloc(sizeof(int) * (levels + 2), st));
  LW_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (levels + 2), st));
  LW_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(WNode) * nr, st));
  int one = 1, zero = 0;
  LW_CUDA_TRY(cudaMemcpyAsync(f0.p, &root_ref, sizeof(int), cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(need.as<int>() + root_ref, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(cnt.p, &one, sizeof(int), cudaMemcpyHostToDevice, st));
  int* cn = cnt.as<int>();
  int* mx = cn + levels + 1;
  for (int L = 0; L < levels; L++) {
    const int* fin = (L & 1) ? f1.as<int>() : f0.as<int>();
    int* fout = (L & 1) ? f0.as<int>() : f1.as<int>();
    k_collapse_level<<<148 * 4, 128, 0, st>>>(bn, fin, cn + L, fout, cn + L + 1, need.as<int>(), out, mx);
  }
  LW_CUDA_TRY(cudaGetLastError());
  int tail[2];
  LW_CUDA_TRY(cudaMemcpyAsync(tail, cn + levels, sizeof(tail), cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  if (tail[0] != 0) {
    set_error("render BVH collapse: frontier not empty after %d levels", levels);
    return LW_ERR_CUDA;
  }
  max_need = tail[1];
  return LW_OK;
}

int alloc_pool(lw_ctx* c, int size) {
  if (c->pool.size == size) return LW_OK;
  free_pool(c);
  Pool& P = c->pool;
  const size_t nvec = 17;  // double2 arrays
  size_t bytes = (size_t)size * (nvec * 16 + 7 * 4 + 1) + 8192;
  size_t got = bytes;
  P.block = take_pool_block(c->device, bytes, got);
  if (!P.block) LW_CUDA_TRY(cudaMalloc(&P.block, bytes));
  c->pool_bytes = got;
  char* p = (char*)P.block;
  auto v2 = [&](double2*& x) {
    x = (double2*)p;
    p += sizeof(double2) * size;
  };
  auto ii = [&](int*& x) {
    x = (int*)p;
    p += sizeof(int) * size;
  };
  v2(P.ray0); v2(P.ray1); v2(P.ray2);
  v2(P.tp0); v2(P.tp1); v2(P.tp2);
  v2(P.misc);
  v2(P.hit0); v2(P.hit1);
  v2(P.sh0); v2(P.sh1); v2(P.sh2); v2(P.sh3); v2(P.sh4);
  v2(P.sh5); v2(P.sh6); v2(P.sh7);
  ii(P.pix); ii(P.flags); ii(P.nprev); ii(P.lpe_state); ii(P.sh_lpe);
  ii(P.q_ext); ii(P.q_shadow);
  P.stage = (unsigned char*)p;
  P.size = size;
  LW_CUDA_TRY(cudaMemsetAsync(P.stage, LW_STAGE_GENERATE, size, c->stream));
  return LW_OK;
}

template <int NODES, bool CMP>
void launch_shadow(lw_ctx* c, cudaStream_t st, int grid, size_t smem, int nr, bool lpe_on, bool count) {
  if (NODES == LW_NODES_GLOBAL ? c->persist_sh : (c->persist_mask & 8) != 0) {
    if (lpe_on)
      k_trace_shadow_p<false, true, NODES, CMP><<<grid, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, c->lpe);
    else if (count)
      k_trace_shadow_p<true, false, NODES, CMP><<<grid, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, c->lpe);
    else
      k_trace_shadow_p<false, false, NODES, CMP><<<grid, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, c->lpe);
    return;
  }
  int use_smem = NODES == LW_NODES_SMEM ? 1 : 0;
  if (lpe_on)
    k_trace_shadow<false, true, NODES, CMP><<<grid, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, use_smem, c->lpe);
  else if (count)
    k_trace_shadow<true, false, NODES, CMP><<<grid, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, use_smem, c->lpe);
  else
    k_trace_shadow<false, false, NODES, CMP><<<grid, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, use_smem, c->lpe);
}

// the instantiated scene classes, most specific first: diffuse + no environment + alias lights
// (Cornell box), diffuse + no environment (light hierarchy), diffuse, alias lights + constant
// environment (layered / glossy materials under a sky colour), alias + no emitters (image
// environment only), any.  k_shade_nee keeps the general kernel for the last two (with the layered
// BSDF its register allocation came out 2-6 registers larger and C4's NEE 4.6 % slower).
#define LW_SCENE_CLASSES_NEE(X) \
  X(LW_MC_DIFFUSE | LW_MC_NOENV | LW_MC_ALIAS) X(LW_MC_DIFFUSE | LW_MC_NOENV) X(LW_MC_DIFFUSE)
#if LW_NEE_L2
#define LW_SCENE_CLASSES_NEE_L2(X) X(LW_MC_ALIAS | LW_MC_ENVCONST | LW_MC_L2) X(LW_MC_ALIAS | LW_MC_NOTRI | LW_MC_L2)
#else
#define LW_SCENE_CLASSES_NEE_L2(X)
#endif
#define LW_SCENE_CLASSES(X) \
  LW_SCENE_CLASSES_NEE(X) X(LW_MC_ALIAS | LW_MC_ENVCONST | LW_MC_L2) X(LW_MC_ALIAS | LW_MC_NOTRI | LW_MC_L2)

// scene class of the wave: the first instantiated class whose properties the scene has
int scene_class(const lw_ctx* c) {
  const DevScene& S = c->S;
  int m = 0;
  if (c->mat_diffuse) m |= LW_MC_DIFFUSE;
  if (S.env_kind == LW_ENV_NONE) m |= LW_MC_NOENV;
  if (S.light_mode != LW_LIGHTS_TREE) m |= LW_MC_ALIAS;
  if (S.nemit == 0) m |= LW_MC_NOTRI;
  if (S.env_kind == LW_ENV_NONE || S.env_kind == LW_ENV_CONSTANT) m |= LW_MC_ENVCONST;
  if (c->mat_max_layers <= 2) m |= LW_MC_L2;
#define LW_SC_PICK(k) \
  if ((m & (k)) == (k)) return (k);
  LW_SCENE_CLASSES(LW_SC_PICK)
#undef LW_SC_PICK
  return LW_MC_ANY;
}

// the two shading kernels for the wave's LPE / light-hierarchy / scene-class configuration (the
// scene classes are instantiated without LPE layers only: wc.mc is LW_MC_ANY when layers are set)
template <bool CMP, int MC>
void launch_shade_nee(lw_ctx* c, cudaStream_t st, int gS, bool lpe_on, bool ltm, size_t ltsm) {
  if (MC == LW_MC_ANY && lpe_on && ltm)
    k_shade_nee<true, true, CMP, LW_MC_ANY><<<gS, 128, ltsm, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
  else if (MC == LW_MC_ANY && lpe_on)
    k_shade_nee<true, false, CMP, LW_MC_ANY><<<gS, 128, 0, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
  else if (ltm)
    k_shade_nee<false, true, CMP, MC><<<gS, 128, ltsm, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
  else
    k_shade_nee<false, false, CMP, MC><<<gS, 128, 0, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
}

template <bool CMP, int MC>
void launch_shade(lw_ctx* c, cudaStream_t st, int gS, bool lpe_on, bool ltm, size_t ltsm) {
  if (MC == LW_MC_ANY && lpe_on && ltm)
    k_shade<true, true, CMP, LW_MC_ANY><<<gS, 128, ltsm, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
  else if (MC == LW_MC_ANY && lpe_on)
    k_shade<true, false, CMP, LW_MC_ANY><<<gS, 128, 0, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
  else if (ltm)
    k_shade<false, true, CMP, MC><<<gS, 128, ltsm, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
  else
    k_shade<false, false, CMP, MC><<<gS, 128, 0, st>>>(c->S, c->pool, c->d_cnt, c->lpe);
}

constexpr int kMaxWaves = 100000;   // a pass that needs more waves is reported as an error

void stamp(lw_ctx* c, cudaStream_t st, const WaveCfg& wc, int stage) {
  if (wc.timed) k_stamp<<<1, 1, 0, st>>>(c->d_stamps, c->d_cnt, stage, kStampCap);
}

// the launches of one wave (wave decision, regeneration / compaction, the four stage kernels,
// wave end), identical on the host-loop path and inside the CUDA-graph loop
template <bool CMP>
void enqueue_wave(lw_ctx* c, cudaStream_t st, const WaveCfg& wc) {
  const lw_render_params& p = c->params;
  const int nr = c->nrnodes;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  const int gT = nsm * 8, gS = nsm * 8, gR = nsm * 4;
  const bool lpe_on = wc.lpe_on, ltm = wc.ltm, count = wc.count, use_smem = wc.use_smem;
  const size_t smem = wc.smem, ltsm = wc.ltsm;
  stamp(c, st, wc, LW_PROF_OTHER);
  k_wave_begin<<<1, 1, 0, st>>>(c->d_cnt, wc.pool, p.regen_fraction, 0, wc.tail_div);
  stamp(c, st, wc, LW_PROF_GENERATE);
  if (lpe_on)
    k_generate<true, CMP><<<gR, 256, 0, st>>>(c->S, c->pool, c->d_fb, c->d_cnt, c->lpe);
  else
    k_generate<false, CMP><<<gR, 256, 0, st>>>(c->S, c->pool, c->d_fb, c->d_cnt, c->lpe);
  stamp(c, st, wc, LW_PROF_TRACE_EXT);
  if (use_smem && (wc.persist_mask & 4)) {
    if (count)
      k_trace_ext_p<true, LW_NODES_SMEM, CMP><<<gT, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr);
    else
      k_trace_ext_p<false, LW_NODES_SMEM, CMP><<<gT, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr);
  } else if (use_smem) {
    if (count)
      k_trace_ext<true, LW_NODES_SMEM, CMP><<<gT, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, 1);
    else
      k_trace_ext<false, LW_NODES_SMEM, CMP><<<gT, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, 1);
  } else {
    if (c->persist && count)
      k_trace_ext_p<true, LW_NODES_GLOBAL, CMP><<<gT, 128, 0, st>>>(c->S, c->pool, c->d_cnt, nr);
    else if (c->persist)
      k_trace_ext_p<false, LW_NODES_GLOBAL, CMP><<<gT, 128, 0, st>>>(c->S, c->pool, c->d_cnt, nr);
    else if (count)
      k_trace_ext<true, LW_NODES_GLOBAL, CMP><<<gT, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, 0);
    else
      k_trace_ext<false, LW_NODES_GLOBAL, CMP><<<gT, 128, smem, st>>>(c->S, c->pool, c->d_cnt, nr, 0);
  }
  stamp(c, st, wc, LW_PROF_SHADE_NEE);
#define LW_SC_NEE(k) \
  case (k): launch_shade_nee<CMP, (k)>(c, st, gS, lpe_on, ltm, ltsm); break;
  switch (wc.mc) {
    LW_SCENE_CLASSES_NEE(LW_SC_NEE)
    LW_SCENE_CLASSES_NEE_L2(LW_SC_NEE)
    default: launch_shade_nee<CMP, LW_MC_ANY>(c, st, gS, lpe_on, ltm, ltsm);
  }
#undef LW_SC_NEE
  stamp(c, st, wc, LW_PROF_SHADE);
#define LW_SC_SHADE(k) \
  case (k): launch_shade<CMP, (k)>(c, st, gS, lpe_on, ltm, ltsm); break;
  switch (wc.mc) {
    LW_SCENE_CLASSES(LW_SC_SHADE)
    default: launch_shade<CMP, LW_MC_ANY>(c, st, gS, lpe_on, ltm, ltsm);
  }
#undef LW_SC_SHADE
  stamp(c, st, wc, LW_PROF_TRACE_SHADOW);
  if (use_smem)
    launch_shadow<LW_NODES_SMEM, CMP>(c, st, gT, smem, nr, lpe_on, count);
  else
    launch_shadow<LW_NODES_GLOBAL, CMP>(c, st, gT, smem, nr, lpe_on, count);
  stamp(c, st, wc, LW_PROF_OTHER);
  k_wave_end<<<1, 1, 0, st>>>(c->d_cnt);
}

// Device-side termination (PAPER.md:599-699 state machine without host round trips): one CUDA
// graph per wave configuration holding a conditional WHILE node whose body is one wave followed by
// k_wave_cond, which keeps the loop running while work is left or paths are alive.  A pass is then
// a handful of stream operations and returns without synchronising.
template <bool CMP>
int build_wave_graph(lw_ctx* c, const WaveCfg& wc) {
  if (c->wave_exec) {
    cudaGraphExecDestroy(c->wave_exec);
    c->wave_exec = nullptr;
  }
  if (!c->cap_stream) LW_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t g;
  LW_CUDA_TRY(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams np = {cudaGraphNodeTypeConditional};
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  if (e == cudaSuccess) e = cudaGraphAddNode(&node, g, nullptr, 0, &np);
  if (e == cudaSuccess)
    e = cudaStreamBeginCaptureToGraph(c->cap_stream, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    enqueue_wave<CMP>(c, c->cap_stream, wc);
    k_wave_cond<<<1, 1, 0, c->cap_stream>>>(c->d_cnt, h, kMaxWaves);
    cudaGraph_t body;
    e = cudaStreamEndCapture(c->cap_stream, &body);
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&c->wave_exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c->wave_exec = nullptr;
    set_error("CUDA graph of the wave loop: %s", cudaGetErrorString(e));
    return LW_ERR_CUDA;
  }
  c->wave_key = wc;
  return LW_OK;
}

// Completes the bookkeeping of the last queued pass: waits for the context stream, then fills the
// per-pass profile (stage times from the timestamps of k_stamp, launches, traversal counters) and
// the running statistics (accumulated on the device by k_stats_accum) from the pinned mirrors.
int pass_fold(lw_ctx* c) {
  if (!c->pass_pending) return LW_OK;
  c->pass_pending = false;
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  const Counters& h = *c->h_cnt;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  c->last_total_ms = ms;
  memset(&c->prof, 0, sizeof(c->prof));
  int64_t launches = c->pass_host_launches + 1;  // + k_stats_accum
  if (c->pass_graph) launches += (int64_t)h.gwaves * 8;  // 7 wave kernels + the loop condition
  if (c->pass_timed) {
    int n = std::min(h.stamp_n, kStampCap);
    launches += n;
    for (int k = 0; k + 1 < n; k++) {
      int sg = (int)(c->h_stamps[k] & 15u);
      if (sg == LW_PROF_END) continue;
      c->prof.stage_ms[sg] += (double)((c->h_stamps[k + 1] >> 4) - (c->h_stamps[k] >> 4)) * 1e-6;
      if (sg != LW_PROF_OTHER) c->prof.stage_launches[sg]++;
    }
  }
  c->prof.total_ms = ms;
  c->prof.kernel_launches = launches;
  c->last_launches = launches;
  c->prof.trace_ext_ms = c->prof.stage_ms[LW_PROF_TRACE_EXT];
  c->prof.trace_shadow_ms = c->prof.stage_ms[LW_PROF_TRACE_SHADOW];
  c->prof.trace_ext_launches = c->prof.stage_launches[LW_PROF_TRACE_EXT];
  c->prof.trace_shadow_launches = c->prof.stage_launches[LW_PROF_TRACE_SHADOW];
  c->prof.pool_slots = c->pool.size;
  c->prof.waves = (int64_t)h.waves;
  c->prof.paths = (int64_t)h.paths;
  c->last_trace_ms = c->prof.trace_ext_ms + c->prof.trace_shadow_ms;
  c->prof.ext_rays = (int64_t)h.rays_ext;
  c->prof.shadow_rays = (int64_t)h.rays_shadow;
  c->prof.ext_nodes = (int64_t)h.ext_nodes;
  c->prof.ext_tris = (int64_t)h.ext_tris;
  c->prof.shadow_nodes = (int64_t)h.sh_nodes;
  c->prof.shadow_tris = (int64_t)h.sh_tris;
  c->prof.shadow_unoccluded = (int64_t)h.sh_unocc;
  c->stats.paths = (int64_t)c->h_acc[0];
  c->stats.rays_extension = (int64_t)c->h_acc[1];
  c->stats.rays_shadow = (int64_t)c->h_acc[2];
  c->stats.nonfinite = (int64_t)c->h_acc[3];
  c->stats.waves = (int64_t)c->h_acc[4];
  c->stats.regenerations = (int64_t)c->h_acc[5];
  if (h.overflow) {
    set_error("wavefront did not terminate");
    return LW_ERR_STATE;
  }
  return LW_OK;
}

template <bool CMP>
int run_pass_t(lw_ctx* c, const WorkRange& w) {
  LW_CHECK_ARG(c->has_scene, "render: no scene uploaded");
  LW_CHECK_ARG(c->configured, "render: lw_render_configure not called");
  // no wait for a previous pass: passes queue on the stream; the profile describes the last one and
  // the running statistics accumulate on the device
  cudaStream_t st = c->stream;
  const lw_render_params& p = c->params;
  int nr = c->nrnodes;
  int use_smem = c->smem_bytes > 0 ? 1 : 0;
  size_t smem = c->smem_bytes;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  Counters zero;
  memset(&zero, 0, sizeof(zero));
  zero.wr = w;
  LW_CUDA_TRY(cudaMemcpyAsync(c->d_cnt, &zero, sizeof(Counters), cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaEventRecord(c->ev0, st));
  long long total = w.nits * w.npix;
  c->pass_graph = false;
  c->pass_timed = false;
  c->pass_host_launches = 0;
  if (p.engine == LW_ENGINE_MEGAKERNEL) {
    int grid = nsm * 8;
    long long need = (total + 127) / 128;
    if (need < grid) grid = (int)std::max<long long>(1, need);
    if (c->lpe.nlayers > 0)
      k_megakernel<true, CMP><<<grid, 128, smem, st>>>(c->S, w, c->d_fb, c->d_cnt, nr, use_smem, c->lpe);
    else
      k_megakernel<false, CMP><<<grid, 128, smem, st>>>(c->S, w, c->d_fb, c->d_cnt, nr, use_smem, c->lpe);
    LW_CUDA_TRY(cudaGetLastError());
    c->pass_host_launches = 1;
  } else {
    WaveCfg wc;
    wc.lpe_on = c->lpe.nlayers > 0;
    wc.ltsm = lt_smem_bytes(c);  // light-hierarchy top staged by the shading kernels
    wc.ltm = wc.ltsm > 0;
    int pool = 1 << p.pool_log2;
    if ((long long)pool > total) {
      long long r = 1;
      while (r < total) r <<= 1;
      pool = (int)std::max<long long>(r, 1024);
    }
    LW_STATUS_TRY(alloc_pool(c, pool));
    wc.pool = pool;
    wc.cmp = CMP;
    wc.use_smem = use_smem;
    wc.smem = smem;
    wc.count = (c->instr & LW_INSTR_COUNT) != 0;
    wc.timed = (c->instr & LW_INSTR_TIME) != 0;
    wc.persist_mask = c->persist_mask;
    wc.tail_div = c->tail_div;
    wc.mc = (c->mat_class_on && !wc.lpe_on) ? scene_class(c) : LW_MC_ANY;
    wc.pool_block = c->pool.block;
    wc.epoch = c->epoch;
    // every slot starts free
    LW_CUDA_TRY(cudaMemsetAsync(c->pool.stage, LW_STAGE_GENERATE, pool, st));
    // the graph is captured when a configuration is used a second time: a context that renders a
    // single pass (one job per context) does not pay the capture / instantiation
    const bool ready = c->wave_exec && c->wave_key == wc;
    const bool graph = c->use_graph && p.megakernel_tail == 0 && (ready || c->last_key == wc);
    c->last_key = wc;
    if (graph) {
      if (!c->wave_exec || !(c->wave_key == wc)) LW_STATUS_TRY(build_wave_graph<CMP>(c, wc));
      LW_CUDA_TRY(cudaGraphLaunch(c->wave_exec, st));
      c->pass_graph = true;
    } else {  // host loop: checks the counters every 8 waves (megakernel tail switch, LW_GRAPH=0)
      const int check_every = 8;
      long long waves = 0;
      for (;;) {
        for (int k = 0; k < check_every; k++) {
          enqueue_wave<CMP>(c, st, wc);
          c->pass_host_launches += 7;
          waves++;
        }
        LW_CUDA_TRY(cudaGetLastError());
        LW_CUDA_TRY(cudaMemcpyAsync(c->h_cnt, c->d_cnt, sizeof(Counters), cudaMemcpyDeviceToHost, st));
        LW_CUDA_TRY(cudaStreamSynchronize(st));
        const Counters& h = *c->h_cnt;
        bool work_left = h.work_next < (unsigned long long)total;
        if (!work_left && h.n_alive == 0) break;
        if (!work_left && p.megakernel_tail > 0 && h.n_alive < p.megakernel_tail) {
          if (wc.lpe_on)
            k_mega_tail<true, CMP><<<nsm * 4, 128, smem, st>>>(c->S, c->pool, c->d_fb, c->d_cnt, nr, use_smem, c->lpe);
          else
            k_mega_tail<false, CMP><<<nsm * 4, 128, smem, st>>>(c->S, c->pool, c->d_fb, c->d_cnt, nr, use_smem, c->lpe);
          k_tail_done<<<1, 1, 0, st>>>(c->d_cnt);
          c->pass_host_launches += 2;
          break;
        }
        if (waves > kMaxWaves) {
          set_error("wavefront did not terminate");
          return LW_ERR_STATE;
        }
      }
    }
    // flush the remaining finished paths
    stamp(c, st, wc, LW_PROF_OTHER);
    k_wave_begin<<<1, 1, 0, st>>>(c->d_cnt, pool, p.regen_fraction, 1, 0);
    stamp(c, st, wc, LW_PROF_GENERATE);
    k_generate<false, CMP><<<nsm * 4, 256, 0, st>>>(c->S, c->pool, c->d_fb, c->d_cnt, c->lpe);
    stamp(c, st, wc, LW_PROF_END);
    c->pass_host_launches += 2;
    c->pass_timed = wc.timed;
  }
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaEventRecord(c->ev1, st));
  k_stats_accum<<<1, 1, 0, st>>>(c->d_cnt, c->d_acc);
  LW_CUDA_TRY(cudaMemcpyAsync(c->h_cnt, c->d_cnt, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(c->h_acc, c->d_acc, sizeof(unsigned long long) * 6, cudaMemcpyDeviceToHost, st));
  if (c->pass_timed && p.engine != LW_ENGINE_MEGAKERNEL)
    LW_CUDA_TRY(cudaMemcpyAsync(c->h_stamps, c->d_stamps, sizeof(unsigned long long) * kStampCap,
                                cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaGetLastError());
  c->pass_pending = true;
  return LW_OK;
}

// NVTX range for profilers (nsys / ncu --nvtx): header-only NVTX v3, free when no tool is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// compressed path state selects the stage-kernel instantiations (no runtime branch in the FP64 ones)
int run_pass(lw_ctx* c, const WorkRange& w) {
  NvtxRange r(c->S.compact ? "lw_render_pass (compact state)" : "lw_render_pass");
  return c->S.compact ? run_pass_t<true>(c, w) : run_pass_t<false>(c, w);
}

}  // namespace

namespace {
// Per-device cache of the fixed context resources (stream, pinned counter mirror, counters,
// events): pinned-host allocation and stream creation cost milliseconds with large variance,
// so a destroyed context returns them for the next one (e.g. one context per progressive job).
struct CtxRes {
  int device;
  cudaStream_t stream;
  Counters *d_cnt, *h_cnt;
  cudaEvent_t ev0, ev1;
  cudaStream_t side;          // scene upload: copies that overlap the BVH build
  cudaEvent_t ev_side0, ev_side1;
};
std::mutex g_res_mu;
std::vector<CtxRes> g_res_free;
constexpr size_t kResCache = 16;

cudaError_t take_res(int device, CtxRes& r) {
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    for (size_t k = 0; k < g_res_free.size(); k++) {
      if (g_res_free[k].device == device) {
        r = g_res_free[k];
        g_res_free.erase(g_res_free.begin() + k);
        return cudaSuccess;
      }
    }
  }
  r.device = device;
  r.stream = nullptr;
  r.d_cnt = r.h_cnt = nullptr;
  r.ev0 = r.ev1 = nullptr;
  r.side = nullptr;
  r.ev_side0 = r.ev_side1 = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&r.d_cnt, kCtrBytes);
  if (e == cudaSuccess) e = cudaMallocHost(&r.h_cnt, kCtrBytes);
  if (e == cudaSuccess) e = cudaEventCreate(&r.ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&r.ev1);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.ev_side0, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.ev_side1, cudaEventDisableTiming);
  return e;
}

void give_res(const CtxRes& r) {
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (g_res_free.size() < kResCache) {
      g_res_free.push_back(r);
      return;
    }
  }
  if (r.d_cnt) cudaFree(r.d_cnt);
  if (r.h_cnt) cudaFreeHost(r.h_cnt);
  if (r.ev0) cudaEventDestroy(r.ev0);
  if (r.ev1) cudaEventDestroy(r.ev1);
  if (r.ev_side0) cudaEventDestroy(r.ev_side0);
  if (r.ev_side1) cudaEventDestroy(r.ev_side1);
  if (r.side) cudaStreamDestroy(r.side);
  if (r.stream) cudaStreamDestroy(r.stream);
}
// NCCL, resolved at first use with dlopen("libnccl.so.2"): in a PyTorch process this is the
// library torch.distributed already loaded; the render library itself has no link-time NCCL
// dependency (stateless kernels and single-GPU rendering never need it).
struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_id)(ncclUniqueId*);
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*destroy)(ncclComm_t);
  const char* (*err)(ncclResult_t);
};

NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_id = (ncclResult_t(*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
    api.init_rank = (ncclResult_t(*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
    api.all_reduce = (ncclResult_t(*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                      cudaStream_t))dlsym(h, "ncclAllReduce");
    api.destroy = (ncclResult_t(*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
    api.err = (const char* (*)(ncclResult_t))dlsym(h, "ncclGetErrorString");
    api.ok = api.get_id && api.init_rank && api.all_reduce && api.destroy && api.err;
  });
  return &api;
}

#define LW_NCCL_TRY(expr)                                                     \
  do {                                                                        \
    ncclResult_t _r = (expr);                                                 \
    if (_r != ncclSuccess) {                                                  \
      set_error("NCCL: %s (%s)", nccl_api()->err(_r), #expr);                 \
      return LW_ERR_CUDA;                                                     \
    }                                                                         \
  } while (0)

// progressive accumulation of a pass: dst += fb, fb = 0 (one read of each, one write of each)
__global__ void k_fb_accumulate(unsigned long long* __restrict__ fb, unsigned long long* __restrict__ dst, long long n,
                                int clear) {
  long long n2 = n >> 1;
  ulonglong2* f2 = reinterpret_cast<ulonglong2*>(fb);
  ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n2; k += (long long)gridDim.x * blockDim.x) {
    ulonglong2 a = f2[k], b = d2[k];
    d2[k] = make_ulonglong2(a.x + b.x, a.y + b.y);
    if (clear) f2[k] = make_ulonglong2(0ull, 0ull);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    dst[n - 1] += fb[n - 1];
    if (clear) fb[n - 1] = 0ull;
  }
}

}  // namespace

extern "C" {

int lw_comm_unique_id(uint8_t* out) {
  LW_CHECK_ARG(out, "null out");
  NcclApi* api = nccl_api();
  if (!api->ok) {
    set_error("NCCL (libnccl.so.2) is not available");
    return LW_ERR_STATE;
  }
  ncclUniqueId id;
  LW_NCCL_TRY(api->get_id(&id));
  static_assert(sizeof(ncclUniqueId) == LW_COMM_ID_BYTES, "ncclUniqueId size");
  memcpy(out, &id, sizeof(id));
  return LW_OK;
}

int lw_ctx_comm_init(lw_ctx* c, const uint8_t* id, int rank, int world) {
  LW_CHECK_ARG(c && id && world >= 1 && rank >= 0 && rank < world, "bad communicator arguments");
  NcclApi* api = nccl_api();
  if (!api->ok) {
    set_error("NCCL (libnccl.so.2) is not available");
    return LW_ERR_STATE;
  }
  cudaSetDevice(c->device);
  if (c->comm) {
    api->destroy(c->comm);
    c->comm = nullptr;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  LW_NCCL_TRY(api->init_rank(&c->comm, world, uid, rank));
  c->comm_rank = rank;
  c->comm_world = world;
  return LW_OK;
}

int lw_framebuffer_reduce(lw_ctx* c) {
  LW_CHECK_ARG(c && c->configured, "not configured");
  if (!c->comm) {
    set_error("lw_framebuffer_reduce: no communicator (lw_ctx_comm_init)");
    return LW_ERR_STATE;
  }
  cudaSetDevice(c->device);
  NvtxRange nv("lw_framebuffer_reduce");
  NcclApi* api = nccl_api();
  LW_NCCL_TRY(api->all_reduce(c->d_fb, c->d_fb, (size_t)(3 * c->fb_pixels), ncclUint64, ncclSum, c->comm, c->stream));
  if (c->lpe.nlayers > 0)
    LW_NCCL_TRY(api->all_reduce(c->lpe.fb, c->lpe.fb, (size_t)(3 * c->lpe.npix * c->lpe.nlayers), ncclUint64, ncclSum,
                                c->comm, c->stream));
  return LW_OK;
}

int lw_framebuffer_accumulate(lw_ctx* c, void* dst, int clear) {
  LW_CHECK_ARG(c && c->configured && dst, "bad arguments");
  LW_CHECK_ARG(((uintptr_t)dst & 15) == 0, "accumulation buffer must be 16-byte aligned");
  cudaSetDevice(c->device);
  long long n = 3 * c->fb_pixels;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  long long need = ((n >> 1) + 255) / 256;
  int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)nsm * 8));
  k_fb_accumulate<<<grid, 256, 0, c->stream>>>(c->d_fb, (unsigned long long*)dst, n, clear);
  LW_CUDA_TRY(cudaGetLastError());
  return LW_OK;
}

int lw_ctx_create(int device, lw_ctx** out) {
  LW_CHECK_ARG(out, "null out");
  LW_CUDA_TRY(cudaSetDevice(device));
  lw_ctx* c = new lw_ctx();
  c->device = device;
  memset(&c->S, 0, sizeof(c->S));
  memset(&c->stats, 0, sizeof(c->stats));
  memset(&c->params, 0, sizeof(c->params));
  memset(&c->prof, 0, sizeof(c->prof));
  // scene, pool and framebuffer memory is stream-ordered from the device's default pool; keep
  // freed blocks reserved so a new context reuses them without driver allocations
  cudaMemPool_t mp;
  if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  CtxRes r;
  cudaError_t e = take_res(device, r);
  if (e != cudaSuccess) {
    give_res(r);
    set_error("context creation failed: %s", cudaGetErrorString(e));
    delete c;
    return LW_ERR_CUDA;
  }
  c->own_stream = c->stream = r.stream;
  c->side_stream = r.side;
  c->ev_side0 = r.ev_side0;
  c->ev_side1 = r.ev_side1;
  c->d_cnt = r.d_cnt;
  c->h_cnt = r.h_cnt;
  c->d_acc = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(r.d_cnt) + kAccOff);
  c->h_acc = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(r.h_cnt) + kAccOff);
  c->d_stamps = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(r.d_cnt) + kStampOff);
  c->h_stamps = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(r.h_cnt) + kStampOff);
  memset(c->h_acc, 0, 64);
  if (cudaMemsetAsync(c->d_acc, 0, 64, c->stream) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) {
    set_error("context creation failed");
    give_res(r);
    delete c;
    return LW_ERR_CUDA;
  }
  c->ev0 = r.ev0;
  c->ev1 = r.ev1;
  *out = c;
  return LW_OK;
}

int lw_ctx_set_stream(lw_ctx* c, void* stream) {
  LW_CHECK_ARG(c, "null ctx");
  LW_STATUS_TRY(pass_fold(c));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->stream = stream ? (cudaStream_t)stream : c->own_stream;
  return LW_OK;
}

int lw_ctx_set_instrumentation(lw_ctx* c, int flags) {
  LW_CHECK_ARG(c, "null ctx");
  c->instr = flags;
  return LW_OK;
}

int lw_ctx_kernel_profile(lw_ctx* c, lw_kernel_profile* out) {
  LW_CHECK_ARG(c && out, "null argument");
  LW_STATUS_TRY(pass_fold(c));
  *out = c->prof;
  return LW_OK;
}

int lw_ctx_destroy(lw_ctx* c) {
  if (!c) return LW_OK;
  cudaSetDevice(c->device);
  pass_fold(c);
  cudaStreamSynchronize(c->stream);
  for (cudaEvent_t e : c->evpool) cudaEventDestroy(e);
  free_scene(c);
  free_pool(c);
  if (c->d_fb) cudaFreeAsync(c->d_fb, c->stream);
  free_lpe(c);
  cudaStreamSynchronize(c->stream);
  if (c->d_qdims) cudaFreeAsync(c->d_qdims, c->stream);
  if (c->d_qperm) cudaFreeAsync(c->d_qperm, c->stream);
  cudaStreamSynchronize(c->stream);
  if (c->comm) nccl_api()->destroy(c->comm);
  if (c->wave_exec) cudaGraphExecDestroy(c->wave_exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  CtxRes r{c->device, c->own_stream, c->d_cnt, c->h_cnt, c->ev0, c->ev1, c->side_stream, c->ev_side0, c->ev_side1};
  give_res(r);
  delete c;
  return LW_OK;
}

int lw_scene_upload(lw_ctx* c, const lw_scene_desc* d) {
  LW_CHECK_ARG(c && d, "null argument");
  NvtxRange nv("lw_scene_upload");
  LW_CHECK_ARG(d->ntris >= 0 && (d->ntris == 0 || (d->verts && d->normals && d->material)), "bad geometry");
  LW_CHECK_ARG(d->nmaterials > 0 && d->materials, "scene needs at least one material");
  LW_CHECK_ARG(d->nemit >= 0 && (d->nemit == 0 || (d->emit_tri && d->emit_radiance && d->emit_twosided && d->emit_weight)),
               "bad emitter arrays");
  cudaSetDevice(c->device);
  LW_STATUS_TRY(pass_fold(c));
  free_scene(c);
  c->epoch++;  // scene pointers are baked into the wave graph
  cudaStream_t st = c->stream;
  DevScene& S = c->S;
  int64_t n = d->ntris;
  c->ntris = n;
  // LW_DEBUG_UPLOAD=1: host wall-clock phases of the upload (stream synchronised) on stderr
  static const bool dbg_up = getenv("LW_DEBUG_UPLOAD") != nullptr;
  auto now_ms = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  auto phase = [&](const char* what, double& t) {
    if (!dbg_up) return;
    cudaStreamSynchronize(st);
    double t1 = now_ms();
    cudaMemPool_t mp;
    uint64_t res = 0, used = 0;
    if (cudaDeviceGetDefaultMemPool(&mp, c->device) == cudaSuccess) {
      cudaMemPoolGetAttribute(mp, cudaMemPoolAttrReservedMemCurrent, &res);
      cudaMemPoolGetAttribute(mp, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    fprintf(stderr, "lw_scene_upload %s %.3f ms (pool reserved %.0f MB, used %.0f MB)\n", what, t1 - t, res / 1e6,
            used / 1e6);
    t = t1;
  };
  double tph = dbg_up ? now_ms() : 0.0;
  for (int64_t k = 0; k < n; k++)
    LW_CHECK_ARG(d->material[k] >= 0 && d->material[k] < d->nmaterials, "material index out of range");
  for (int64_t e = 0; e < d->nemit; e++) LW_CHECK_ARG(d->emit_tri[e] >= 0 && d->emit_tri[e] < n, "emitter triangle out of range");
  double* dv;
  LW_STATUS_TRY(dev_upload(c, dv, d->verts, 9 * n));
  // Copies the BVH build does not need (shading normals, environment image and texel weights) run
  // on the context's side stream and overlap the build; the main stream waits for them before the
  // environment tables (and, through `side_done`, before any exit path frees a buffer).
  const bool env_img = d->env_kind == LW_ENV_IMAGE && d->env_width > 0 && d->env_height > 0 && d->env_image &&
                       d->env_weight;
  const int64_t env_nt = env_img ? (int64_t)d->env_width * d->env_height : 0;
  double* dn;
  LW_STATUS_TRY(dev_alloc(c, dn, 9 * n));
  float* env_dimg = nullptr;
  DevBuf env_wbuf;  // texel weights: scratch, freed once the tables are built
  if (env_img) {
    LW_STATUS_TRY(dev_alloc(c, env_dimg, 3 * env_nt));
    LW_CUDA_TRY(env_wbuf.alloc(sizeof(double) * env_nt, st));
  }
  LW_CUDA_TRY(cudaEventRecord(c->ev_side0, st));  // allocations ordered before the side copies
  LW_CUDA_TRY(cudaStreamWaitEvent(c->side_stream, c->ev_side0, 0));
  if (n > 0) LW_CUDA_TRY(cudaMemcpyAsync(dn, d->normals, sizeof(double) * 9 * n, cudaMemcpyHostToDevice, c->side_stream));
  if (env_img) {
    LW_CUDA_TRY(cudaMemcpyAsync(env_dimg, d->env_image, sizeof(float) * 3 * env_nt, cudaMemcpyHostToDevice, c->side_stream));
    LW_CUDA_TRY(cudaMemcpyAsync(env_wbuf.p, d->env_weight, sizeof(double) * env_nt, cudaMemcpyHostToDevice, c->side_stream));
  }
  LW_CUDA_TRY(cudaEventRecord(c->ev_side1, c->side_stream));
  struct SideDone {  // main stream waits for the side copies on every exit (before env_wbuf's free)
    lw_ctx* c;
    ~SideDone() { cudaStreamWaitEvent(c->stream, c->ev_side1, 0); }
  } side_done{c};
  int* dm;
  LW_STATUS_TRY(dev_upload(c, dm, (const int*)d->material, n));
  lw_material* dmat;
  LW_STATUS_TRY(dev_upload(c, dmat, d->materials, d->nmaterials));
  c->mat_diffuse = true;
  c->mat_max_layers = 0;
  for (int k = 0; k < d->nmaterials; k++) {
    const lw_material& m = d->materials[k];
    if (!(m.nlayers == 1 && m.layers[0].kind == LW_BSDF_DIFFUSE && m.layers[0].coat == 0)) c->mat_diffuse = false;
    c->mat_max_layers = std::max(c->mat_max_layers, (int)m.nlayers);
  }
  S.verts = dv;
  S.normals = dn;
  S.material = dm;
  S.materials = dmat;
  phase("validate+copy", tph);
  // the reference-layout median tree (geometry.py:100-148 arrays) is built here only when it is
  // the render tree; otherwise on demand by lw_ctx_bvh_info / lw_ctx_bvh_download
  c->ref_built = false;
  // render tree: the requested kind; a SAH tree whose worst path would overflow the traversal
  // stack (pathological, e.g. exponentially spaced triangles) is replaced by the median tree
  // (depth <= 2 + log2 n).  Hits do not depend on the tree, so the image is unchanged.
  int kind = d->bvh_kind;
  int nr = 0, levels = 0, root_ref = leaf_ref(0, 0);
  LTri* lt;
  WNode* wn = nullptr;
  double rb[6] = {0, 0, 0, 0, 0, 0};
  LW_STATUS_TRY(dev_alloc(c, lt, n > 0 ? n : 1));
  for (;;) {
  SahNode* bn = nullptr;  // binary tree (FP64 child boxes), collapsed to the 4-wide layout below
  if (kind == LW_BVH_MEDIAN) {
    if (!c->ref_built) {
      LW_STATUS_TRY(bvh_build_device(dv, n, st, c->ref_bvh));
      c->ref_built = true;
    }
    int64_t nn = c->ref_bvh.nnodes;
    // render layout derived from the median tree on the device
    nr = nrnodes_of(c);
    LW_CUDA_TRY(cudaMallocAsync(&bn, sizeof(SahNode) * (nr > 0 ? nr : 1), st));
    if (n > 0) {
      int* flag;
      int* imap;
      LW_STATUS_TRY(dev_alloc(c, flag, nn));
      LW_STATUS_TRY(dev_alloc(c, imap, nn));
      k_internal_flags<<<grid_for(nn, 256, 1 << 30), 256, 0, st>>>(c->ref_bvh.children, nn, flag);
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, imap, (int)nn, st);
      void* tmp;
      LW_CUDA_TRY(cudaMallocAsync(&tmp, tb > 0 ? tb : 16, st));
      LW_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flag, imap, (int)nn, st));
      k_build_rnodes<<<grid_for(nn, 256, 1 << 30), 256, 0, st>>>(c->ref_bvh.bounds, c->ref_bvh.children, nn, imap, bn);
      k_build_ltris<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(dv, c->ref_bvh.order, n, lt);
      LW_CUDA_TRY(cudaGetLastError());
      LW_CUDA_TRY(cudaStreamSynchronize(st));
      cudaFreeAsync(tmp, st);
    }
    long long rc[2] = {-1, 0};
    LW_CUDA_TRY(cudaMemcpyAsync(rb, c->ref_bvh.bounds, sizeof(rb), cudaMemcpyDeviceToHost, st));
    LW_CUDA_TRY(cudaMemcpyAsync(rc, c->ref_bvh.children, sizeof(rc), cudaMemcpyDeviceToHost, st));
    LW_CUDA_TRY(cudaStreamSynchronize(st));
    root_ref = rc[0] >= 0 ? 0 : (int)(-(1 + ((-(rc[0] + 1)) << 3 | rc[1])));
    levels = 2;  // median split: depth <= 2 + log2(n)
    while ((1LL << (levels - 2)) < n) levels++;
  } else {
    // binned-SAH render tree built on the device (lw_sah_build.cu)
    DeviceSah ds;
    int rc_sah = sah_build_device(dv, n, st, ds);
    if (rc_sah != LW_OK) {
      if (ds.nodes) cudaFreeAsync(ds.nodes, st);
      if (ds.order) cudaFreeAsync(ds.order, st);
      return rc_sah;
    }
    nr = (int)ds.nnodes;
    bn = ds.nodes;
    if (n > 0) k_build_ltris_i32<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(dv, ds.order, n, lt);
    LW_CUDA_TRY(cudaGetLastError());
    LW_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFreeAsync(ds.order, st);
    for (int a = 0; a < 6; a++) rb[a] = ds.root_box[a];
    root_ref = ds.root_ref;
    levels = ds.levels;
  }
  LW_STATUS_TRY(dev_alloc(c, wn, nr > 0 ? nr : 1));
  int max_need = 0;
  phase("binary-tree", tph);
  int rc_w = collapse_wide(c, bn, nr, root_ref, levels, wn, max_need);
  if (bn) cudaFreeAsync(bn, st);
  LW_STATUS_TRY(rc_w);
  if (getenv("LW_DEBUG_STACK")) fprintf(stderr, "render BVH kind %d: %d wide nodes, stack need %d\n", kind, nr, max_need);
  if (max_need <= LW_STACK) break;
  if (kind != LW_BVH_MEDIAN) {
    kind = LW_BVH_MEDIAN;
    continue;
  }
  set_error("render BVH too deep: a path needs %d traversal stack entries (limit %d)", max_need, LW_STACK);
  return LW_ERR_INVALID;
  }
  phase("collapse", tph);
  c->nrnodes = nr;
  S.bvh.nodes = wn;
  S.bvh.tris = lt;
  S.bvh.ntris = n;
  S.bvh.root_ref = root_ref;
  for (int a = 0; a < 6; a++) S.bvh.root_box[a] = rb[a];
  for (int a = 0; a < 3; a++) S.bvh.absmax[a] = std::max(fabs(rb[a]), fabs(rb[3 + a]));
  // stage in shared memory when the whole render BVH fits comfortably
  S.bvh.nstride = (int)sizeof(WNode);
  size_t bytes = smem_bvh_bytes(nr, n);
  c->smem_bytes = (n > 0 && bytes <= 48 * 1024) ? bytes : 0;
  // emitters
  int* eot;
  LW_STATUS_TRY(dev_alloc(c, eot, n > 0 ? n : 1));
  LW_CUDA_TRY(cudaMemsetAsync(eot, 0xff, sizeof(int) * (n > 0 ? n : 1), st));
  S.emit_of_tri = eot;
  S.nemit = d->nemit;
  if (d->nemit > 0) {
    std::vector<double> prob(d->nemit), pdf(d->nemit);
    std::vector<int32_t> alias(d->nemit);
    if (alias_build(d->emit_weight, d->nemit, prob.data(), alias.data(), pdf.data()) != LW_OK) {
      S.nemit = 0;  // no light carries energy (oracle: same rule)
    }
    long long* et;
    double *er, *ea, *ep, *epdf;
    int *e2, *eal;
    LW_STATUS_TRY(dev_upload(c, et, (const long long*)d->emit_tri, d->nemit));
    LW_STATUS_TRY(dev_upload(c, er, d->emit_radiance, 3 * d->nemit));
    LW_STATUS_TRY(dev_upload(c, e2, (const int*)d->emit_twosided, d->nemit));
    LW_STATUS_TRY(dev_alloc(c, ea, d->nemit));
    LW_STATUS_TRY(dev_upload(c, ep, prob.data(), d->nemit));
    LW_STATUS_TRY(dev_upload(c, epdf, pdf.data(), d->nemit));
    LW_STATUS_TRY(dev_upload(c, eal, (const int*)alias.data(), d->nemit));
    k_emitters<<<grid_for(d->nemit, 256, 1 << 30), 256, 0, st>>>(dv, et, d->nemit, ea, eot);
    LW_CUDA_TRY(cudaGetLastError());
    S.emit_tri = et;
    S.emit_rad = er;
    S.emit_two = e2;
    S.emit_area = ea;
    S.emit_prob = ep;
    S.emit_pdf = epdf;
    S.emit_alias = eal;
    LW_CUDA_TRY(cudaStreamSynchronize(st));
  }
  // light hierarchy, built on the host like the alias tables
  S.light_mode = LW_LIGHTS_ALIAS;
  memset(&S.lt, 0, sizeof(S.lt));
  S.lt_nheap = 0;
  c->lt_dfs.clear();
  c->lt_path.clear();
  c->lt_depth.clear();
  if ((d->light_sampler & LW_LIGHTS_TREE) && S.nemit > 0) {
    std::vector<LwLightNode> ln;
    std::vector<unsigned long long> lp;
    std::vector<int> ld;
    LW_STATUS_TRY(light_tree_build(d->verts, d->emit_tri, d->emit_weight, d->emit_twosided, d->nemit, ln, lp, ld));
    // heap order for the device (children 2i+1, 2i+2): the top levels become a contiguous prefix
    int dmax = 0;
    for (int v : ld) dmax = std::max(dmax, v);
    LW_CHECK_ARG(dmax <= 26, "light tree too deep for the heap layout (more than 2^26 emitters)");
    int64_t nheap = (2LL << dmax) - 1;
    std::vector<LwLightNode> hp(nheap);
    std::vector<std::pair<int64_t, int64_t>> todo{{0, 0}};  // (dfs id, heap id)
    while (!todo.empty()) {
      auto [di, hi] = todo.back();
      todo.pop_back();
      hp[hi] = ln[di];
      if (ln[di].right >= 0) {
        todo.push_back({ln[di].right, 2 * hi + 2});
        todo.push_back({di + 1, 2 * hi + 1});
        hp[hi].right = 1;
      }
    }
    LwLightNode* dn;
    unsigned long long* dp;
    int* dd;
    LW_STATUS_TRY(dev_upload(c, dn, hp.data(), nheap));
    LW_STATUS_TRY(dev_upload(c, dp, lp.data(), (int64_t)lp.size()));
    LW_STATUS_TRY(dev_upload(c, dd, ld.data(), (int64_t)ld.size()));
    LW_CUDA_TRY(cudaStreamSynchronize(st));  // host vectors go out of scope
    S.lt.nodes = dn;
    S.lt.top = dn;
    S.lt.ntop = 0;
    S.lt.path = dp;
    S.lt.depth = dd;
    S.lt_nheap = (int)nheap;
    S.light_mode = LW_LIGHTS_TREE;
    c->lt_nodes = (int64_t)ln.size();
    c->lt_dfs = std::move(ln);
    c->lt_path = std::move(lp);
    c->lt_depth = std::move(ld);
  }
  // environment
  S.env_kind = d->env_kind;
  S.env_w = d->env_width;
  S.env_h = d->env_height;
  for (int k = 0; k < 3; k++) S.env_const[k] = d->env_constant[k];
  S.env_scale = d->env_scale;
  if (d->env_kind == LW_ENV_IMAGE) {
    LW_CHECK_ARG(d->env_width > 0 && d->env_height > 0 && d->env_image && d->env_weight, "bad environment image");
    int64_t nt = (int64_t)d->env_width * d->env_height;
    const int W = d->env_width, H = d->env_height;
    float* img = env_dimg;  // copied on the side stream at the start of the upload
    double *dw, *pp, *pd, *rp;
    int *pa, *ra;
    LW_STATUS_TRY(dev_alloc(c, pp, nt));
    LW_STATUS_TRY(dev_alloc(c, pd, nt));
    LW_STATUS_TRY(dev_alloc(c, pa, nt));
    LW_STATUS_TRY(dev_alloc(c, rp, H));
    LW_STATUS_TRY(dev_alloc(c, ra, H));
    // worklists are scratch: freed (stream-ordered) once the tables are built
    DevBuf bs, bl, brs, brp, bbad;
    LW_CUDA_TRY(bs.alloc(sizeof(int) * nt, st));
    LW_CUDA_TRY(bl.alloc(sizeof(int) * nt, st));
    LW_CUDA_TRY(brs.alloc(sizeof(double) * H, st));
    LW_CUDA_TRY(brp.alloc(sizeof(double) * H, st));
    LW_CUDA_TRY(bbad.alloc(sizeof(int), st));
    dw = env_wbuf.as<double>();
    LW_CUDA_TRY(cudaStreamWaitEvent(st, c->ev_side1, 0));  // image and weights are on the device
    // per-table thread blocks in shared memory when a row / the marginal fits (W, H <= 16384);
    // LW_ENV_SERIAL=1 (or larger images) keeps the one-thread-per-row form -- identical tables
    static const bool env_serial = getenv("LW_ENV_SERIAL") != nullptr;
    const size_t row_smem = (size_t)W * 12, col_smem = (size_t)H * 12;
    if (!env_serial && row_smem <= 192 * 1024 && col_smem <= 192 * 1024) {
      const int mx = (int)std::max(row_smem, col_smem);
      LW_CUDA_TRY(cudaFuncSetAttribute(k_env_rows_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      LW_CUDA_TRY(cudaFuncSetAttribute(k_env_marginal_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      int nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
      k_env_rows_blk<<<std::min(H, nsm * 8), kAliasThreads, row_smem, st>>>(dw, W, H, pp, pa, pd, brs.as<double>());
      k_env_marginal_blk<<<1, kAliasThreads, col_smem, st>>>(brs.as<double>(), H, rp, ra, brp.as<double>(), bbad.as<int>());
    } else {
      k_env_rows<<<(H + 63) / 64, 64, 0, st>>>(dw, W, H, pp, pa, pd, brs.as<double>(), bs.as<int>(), bl.as<int>());
      k_env_marginal<<<1, 1, 0, st>>>(brs.as<double>(), H, rp, ra, brp.as<double>(), bs.as<int>(), bl.as<int>(),
                                      bbad.as<int>());
    }
    k_env_pdf<<<grid_for(nt, 256, 148 * 16), 256, 0, st>>>(pd, brp.as<double>(), W, nt);
    LW_CUDA_TRY(cudaGetLastError());
    int bad = 1;
    LW_CUDA_TRY(cudaMemcpyAsync(&bad, bbad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    LW_CUDA_TRY(cudaStreamSynchronize(st));
    if (bad) {
      S.env_kind = LW_ENV_NONE;
    } else {
      S.env_img = img;
      S.env_prob = pp;
      S.env_pdf = pd;
      S.env_alias = pa;
      S.env_rprob = rp;
      S.env_ralias = ra;
    }
  }
  if (d->env_kind != LW_ENV_IMAGE && d->env_kind != LW_ENV_CONSTANT) S.env_kind = LW_ENV_NONE;
  S.env_mode = 0;
  memset(&S.env_pyr, 0, sizeof(S.env_pyr));
  if (S.env_kind == LW_ENV_IMAGE && (d->light_sampler & LW_LIGHTS_ENV_PYRAMID)) {
    std::vector<double> lvl, top;
    LwEnvPyr ep;
    LW_STATUS_TRY(env_pyramid_build(d->env_width, d->env_height, d->env_weight, lvl, top, ep));
    double *dl, *dt;
    LW_STATUS_TRY(dev_upload(c, dl, lvl.data(), (int64_t)lvl.size()));
    LW_STATUS_TRY(dev_upload(c, dt, top.data(), (int64_t)top.size()));
    LW_CUDA_TRY(cudaStreamSynchronize(st));  // host vectors go out of scope
    ep.lvl = dl;
    ep.top = dt;
    S.env_pyr = ep;
    S.env_mode = LW_LIGHTS_ENV_PYRAMID;
  }
  bool has_env = S.env_kind != LW_ENV_NONE, has_tri = S.nemit > 0;
  S.p_env = has_env ? (has_tri ? d->p_env : 1.0) : 0.0;
  S.p_tri = has_tri ? (has_env ? 1.0 - d->p_env : 1.0) : 0.0;
  for (int k = 0; k < 3; k++) {
    S.cam_pos[k] = d->cam_pos[k];
    S.cam_fwd[k] = d->cam_fwd[k];
    S.cam_right[k] = d->cam_right[k];
    S.cam_up[k] = d->cam_up[k];
  }
  S.tan_half = d->tan_half_fov;
  LW_CUDA_TRY(cudaStreamWaitEvent(st, c->ev_side1, 0));  // shading normals (and the environment) landed
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  phase("lights+env", tph);
  c->has_scene = true;
  return LW_OK;
}

int lw_render_configure(lw_ctx* c, const lw_render_params* p) {
  LW_CHECK_ARG(c && p, "null argument");
  LW_CHECK_ARG(p->width > 0 && p->height > 0, "resolution must be positive");
  LW_CHECK_ARG((int64_t)p->width * p->height < (1LL << 31), "resolution too large");
  LW_CHECK_ARG(p->max_depth >= 1 && p->max_depth <= 255, "max_depth must be in [1, 255]");
  LW_CHECK_ARG(p->engine == LW_ENGINE_WAVEFRONT || p->engine == LW_ENGINE_MEGAKERNEL, "unknown engine");
  LW_CHECK_ARG(p->pool_log2 >= 10 && p->pool_log2 <= 26, "pool_log2 must be in [10, 26]");
  LW_CHECK_ARG(p->estimator >= LW_EST_MIS && p->estimator <= LW_EST_BSDF, "unknown estimator");
  LW_CHECK_ARG(p->ndims >= 4 + 8 * (int64_t)p->max_depth, "dimension table too small for max_depth");
  cudaSetDevice(c->device);
  std::vector<QmcDim> dims;
  std::vector<uint16_t> perm;
  LW_STATUS_TRY(pack_qmc_tables(p->bases, p->ndims, p->perm_flat, p->perm_len, p->perm_offset, dims, perm));
  if (c->d_qdims) cudaFreeAsync(c->d_qdims, c->stream);
  if (c->d_qperm) cudaFreeAsync(c->d_qperm, c->stream);
  c->d_qdims = nullptr;
  c->d_qperm = nullptr;
  LW_CUDA_TRY(cudaMallocAsync(&c->d_qdims, sizeof(QmcDim) * dims.size(), c->stream));
  LW_CUDA_TRY(cudaMallocAsync(&c->d_qperm, sizeof(uint16_t) * perm.size(), c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(c->d_qdims, dims.data(), sizeof(QmcDim) * dims.size(), cudaMemcpyHostToDevice, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(c->d_qperm, perm.data(), sizeof(uint16_t) * perm.size(), cudaMemcpyHostToDevice, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));  // host vectors go out of scope
  c->epoch++;
  c->params = *p;
  c->params.bases = nullptr;
  c->params.perm_flat = nullptr;
  c->params.perm_offset = nullptr;
  c->S.qdims = c->d_qdims;
  c->S.qperm = c->d_qperm;
  c->S.W = p->width;
  c->S.H = p->height;
  c->S.max_depth = p->max_depth;
  c->S.rr_start = p->rr_start;
  c->S.estimator = p->estimator;
  c->S.compact = p->compact_state != 0;
  int64_t px = (int64_t)p->width * p->height;
  if (px != c->fb_pixels) {
    free_lpe(c);  // layer framebuffers have the old size
    if (c->d_fb) cudaFreeAsync(c->d_fb, c->stream);
    c->d_fb = nullptr;
    LW_CUDA_TRY(cudaMallocAsync(&c->d_fb, sizeof(unsigned long long) * 3 * px, c->stream));
    c->fb_pixels = px;
    LW_CUDA_TRY(cudaMemsetAsync(c->d_fb, 0, sizeof(unsigned long long) * 3 * px, c->stream));
  }
  c->configured = true;
  return LW_OK;
}

int lw_framebuffer_clear(lw_ctx* c) {
  LW_CHECK_ARG(c && c->configured, "not configured");
  LW_STATUS_TRY(pass_fold(c));
  LW_CUDA_TRY(cudaMemsetAsync(c->d_acc, 0, 64, c->stream));
  memset(c->h_acc, 0, 64);
  LW_CUDA_TRY(cudaMemsetAsync(c->d_fb, 0, sizeof(unsigned long long) * 3 * c->fb_pixels, c->stream));
  if (c->lpe.nlayers > 0)
    LW_CUDA_TRY(cudaMemsetAsync(c->lpe.fb, 0, sizeof(unsigned long long) * 3 * c->lpe.npix * c->lpe.nlayers, c->stream));
  memset(&c->stats, 0, sizeof(c->stats));
  return LW_OK;
}

int lw_render_pass(lw_ctx* c, int64_t it_begin, int64_t it_end) {
  LW_CHECK_ARG(c && c->configured, "not configured");
  return lw_render_pass_pixels(c, it_begin, it_end, 0, c->fb_pixels);
}

int lw_render_pass_pixels(lw_ctx* c, int64_t it_begin, int64_t it_end, int64_t pix_begin, int64_t pix_end) {
  LW_CHECK_ARG(c && c->configured, "not configured");
  LW_CHECK_ARG(it_begin >= 0 && it_end >= it_begin, "bad iteration range");
  LW_CHECK_ARG(pix_begin >= 0 && pix_end <= c->fb_pixels && pix_end >= pix_begin, "bad pixel range");
  if (it_end == it_begin || pix_end == pix_begin) return LW_OK;
  // qmc.py:194-195: the global sample index must fit in 64 bits (here: in a signed int64)
  unsigned __int128 maxidx = (unsigned __int128)(it_end - 1) * (unsigned __int128)c->fb_pixels + (unsigned __int128)pix_end;
  if (maxidx >> 63) {
    set_error("sample index exceeds 64 bits");
    return LW_ERR_OVERFLOW;
  }
  cudaSetDevice(c->device);
  WorkRange w{it_begin, it_end - it_begin, pix_begin, pix_end - pix_begin, 0, 1, 1, 1};
  // whole frames are enumerated in tiles of 32 items: 8x4 pixels, or with LW_TILE_ITS = 2 / 4 / 8
  // iterations of 4x4 / 4x2 / 2x2 pixels (LW_TILES=0: row order); the sample index of a
  // (pixel, iteration) -- hence the image -- does not depend on the order
  static const bool tiles = getenv("LW_TILES") ? atoi(getenv("LW_TILES")) != 0 : true;
  static const int tis = getenv("LW_TILE_ITS") ? atoi(getenv("LW_TILE_ITS")) : 8;
  int ti = (tis == 1 || tis == 2 || tis == 4 || tis == 8 || tis == 16 || tis == 32) ? tis : 8;
  while (ti > 1 && (it_end - it_begin) % ti != 0) ti >>= 1;  // the pass's iterations split into blocks
  static const int tws[6] = {8, 4, 4, 2, 2, 1};  // tile width for ti = 1, 2, 4, 8, 16, 32
  const int tw = tws[__builtin_ctz(ti)], th = 32 / (ti * tw);
  if (tiles && pix_begin == 0 && pix_end == c->fb_pixels && c->params.width % tw == 0 &&
      c->params.height % th == 0 && (it_end - it_begin) % ti == 0) {
    w.tiles_x = c->params.width / tw;
    w.tw = tw;
    w.th = th;
    w.ti = ti;
  }
  return run_pass(c, w);
}

int lw_ctx_synchronize(lw_ctx* c) {
  LW_CHECK_ARG(c, "null ctx");
  LW_STATUS_TRY(pass_fold(c));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_framebuffer_download(lw_ctx* c, int64_t* host_fb) {
  LW_CHECK_ARG(c && c->configured && host_fb, "bad arguments");
  LW_CUDA_TRY(cudaMemcpyAsync(host_fb, c->d_fb, sizeof(int64_t) * 3 * c->fb_pixels, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_framebuffer_resolve(lw_ctx* c, double inv_samples, float* host_rgb) {
  LW_CHECK_ARG(c && c->configured && host_rgb, "bad arguments");
  long long n = 3 * c->fb_pixels;
  float* d_out;
  LW_CUDA_TRY(cudaMallocAsync((void**)&d_out, sizeof(float) * n, c->stream));
  double scale = inv_samples / 1048576.0;
  k_resolve<<<grid_for(n, 256, 1 << 30), 256, 0, c->stream>>>(c->d_fb, n, scale, d_out);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(host_rgb, d_out, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaFreeAsync(d_out, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_framebuffer_copy_device(lw_ctx* c, void* dst) {
  LW_CHECK_ARG(c && c->configured && dst, "bad arguments");
  LW_CUDA_TRY(cudaMemcpyAsync(dst, c->d_fb, sizeof(int64_t) * 3 * c->fb_pixels, cudaMemcpyDeviceToDevice, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_framebuffer_upload(lw_ctx* c, const int64_t* host_fb) {
  LW_CHECK_ARG(c && c->configured && host_fb, "bad arguments");
  LW_CUDA_TRY(cudaMemcpyAsync(c->d_fb, host_fb, sizeof(int64_t) * 3 * c->fb_pixels, cudaMemcpyHostToDevice, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_framebuffer_load_device(lw_ctx* c, const void* src) {
  LW_CHECK_ARG(c && c->configured && src, "bad arguments");
  LW_CUDA_TRY(cudaMemcpyAsync(c->d_fb, src, sizeof(int64_t) * 3 * c->fb_pixels, cudaMemcpyDeviceToDevice, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_get_stats(lw_ctx* c, lw_render_stats* s) {
  LW_CHECK_ARG(c && s, "null argument");
  LW_STATUS_TRY(pass_fold(c));
  *s = c->stats;
  return LW_OK;
}

int lw_ctx_last_pass_timing(lw_ctx* c, double* trace_ms, double* total_ms, int64_t* launches) {
  LW_CHECK_ARG(c, "null ctx");
  LW_STATUS_TRY(pass_fold(c));
  if (trace_ms) *trace_ms = c->last_trace_ms;
  if (total_ms) *total_ms = c->last_total_ms;
  if (launches) *launches = c->last_launches;
  return LW_OK;
}

static int dbg_rays(lw_ctx* c, const double* o, const double* d, const double* tm, int64_t n, DevBuf& bo, DevBuf& bd,
                    DevBuf& bt) {
  LW_CUDA_TRY(bo.alloc(sizeof(double) * 3 * n));
  LW_CUDA_TRY(bd.alloc(sizeof(double) * 3 * n));
  LW_CUDA_TRY(bt.alloc(sizeof(double) * n));
  LW_CUDA_TRY(cudaMemcpyAsync(bo.p, o, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(bd.p, d, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(bt.p, tm, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  return LW_OK;
}

int lw_ctx_trace_closest(lw_ctx* c, const double* o, const double* d, const double* tm, int64_t n, double* out_t,
                         int64_t* out_tri, double* out_bary) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  if (n <= 0) return LW_OK;
  cudaSetDevice(c->device);
  DevBuf bo, bd, bt, rt, rtri, rb;
  LW_STATUS_TRY(dbg_rays(c, o, d, tm, n, bo, bd, bt));
  LW_CUDA_TRY(rt.alloc(sizeof(double) * n));
  LW_CUDA_TRY(rtri.alloc(sizeof(long long) * n));
  LW_CUDA_TRY(rb.alloc(sizeof(double) * 2 * n));
  k_trace_closest_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, c->stream>>>(c->S, bo.as<double>(), bd.as<double>(),
                                                                         bt.as<double>(), n, rt.as<double>(),
                                                                         rtri.as<long long>(), rb.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_t, rt.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_tri, rtri.p, sizeof(long long) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_bary, rb.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_ctx_trace_any(lw_ctx* c, const double* o, const double* d, const double* tm, int64_t n, int32_t* occ) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  if (n <= 0) return LW_OK;
  cudaSetDevice(c->device);
  DevBuf bo, bd, bt, ro;
  LW_STATUS_TRY(dbg_rays(c, o, d, tm, n, bo, bd, bt));
  LW_CUDA_TRY(ro.alloc(sizeof(int) * n));
  k_trace_any_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, c->stream>>>(c->S, bo.as<double>(), bd.as<double>(),
                                                                     bt.as<double>(), n, ro.as<int>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(occ, ro.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_ctx_camera_rays(lw_ctx* c, const int64_t* idx, int64_t n, double* out_o, double* out_d) {
  LW_CHECK_ARG(c && c->has_scene && c->configured, "scene and configuration required");
  if (n <= 0) return LW_OK;
  cudaSetDevice(c->device);
  DevBuf bi, bo, bd;
  LW_CUDA_TRY(bi.alloc(sizeof(long long) * n));
  LW_CUDA_TRY(bo.alloc(sizeof(double) * 3 * n));
  LW_CUDA_TRY(bd.alloc(sizeof(double) * 3 * n));
  LW_CUDA_TRY(cudaMemcpyAsync(bi.p, idx, sizeof(long long) * n, cudaMemcpyHostToDevice, c->stream));
  k_camera_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, c->stream>>>(c->S, bi.as<long long>(), n, bo.as<double>(),
                                                                  bd.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_o, bo.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_d, bd.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

static int ensure_ref_bvh(lw_ctx* c) {
  if (c->ref_built) return LW_OK;
  LW_STATUS_TRY(bvh_build_device(c->S.verts, c->ntris, c->stream, c->ref_bvh));
  c->ref_built = true;
  return LW_OK;
}

int lw_ctx_bvh_info(lw_ctx* c, int64_t* nnodes) {
  LW_CHECK_ARG(c && c->has_scene && nnodes, "no scene");
  LW_STATUS_TRY(ensure_ref_bvh(c));
  *nnodes = c->ref_bvh.nnodes;
  return LW_OK;
}

int lw_ctx_bvh_download(lw_ctx* c, double* bounds, int64_t* children, int64_t* order) {
  LW_CHECK_ARG(c && c->has_scene && bounds && children, "no scene");
  LW_STATUS_TRY(ensure_ref_bvh(c));
  int64_t nn = c->ref_bvh.nnodes;
  LW_CUDA_TRY(cudaMemcpyAsync(bounds, c->ref_bvh.bounds, sizeof(double) * 6 * nn, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(children, c->ref_bvh.children, sizeof(long long) * 2 * nn, cudaMemcpyDeviceToHost, c->stream));
  if (c->ntris > 0 && order)
    LW_CUDA_TRY(cudaMemcpyAsync(order, c->ref_bvh.order, sizeof(long long) * c->ntris, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_ctx_light_tree_info(lw_ctx* c, int64_t* nnodes) {
  LW_CHECK_ARG(c && c->has_scene && nnodes, "no scene");
  *nnodes = c->lt_nodes;
  return LW_OK;
}

int lw_ctx_light_tree_download(lw_ctx* c, double* nodes15, int32_t* right, uint64_t* path, int32_t* depth) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  if (c->lt_nodes == 0) return LW_OK;
  const std::vector<LwLightNode>& h = c->lt_dfs;
  for (size_t k = 0; k < h.size(); k++) {
    double* o = nodes15 ? nodes15 + 15 * k : nullptr;
    if (o) {
      for (int a = 0; a < 3; a++) {
        o[a] = h[k].lo[a];
        o[3 + a] = h[k].hi[a];
      }
      o[6] = h[k].tot;
      for (int b = 0; b < 8; b++) o[7 + b] = h[k].flux[b];
    }
    if (right) right[k] = h[k].right;
  }
  for (int64_t e = 0; e < c->S.nemit; e++) {
    if (path) path[e] = c->lt_path[e];
    if (depth) depth[e] = c->lt_depth[e];
  }
  return LW_OK;
}

int lw_ctx_light_sample(lw_ctx* c, const double* x, const double* nrm, const double* u, int64_t n, int64_t* out_e,
                        double* out_psel, double* out_u) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  LW_CHECK_ARG(c->lt_nodes > 0, "the scene has no light hierarchy (pack_scene(..., lights='tree'))");
  if (n <= 0) return LW_OK;
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  DevBuf bx, bn, bu, be, bp, bo;
  LW_CUDA_TRY(bx.alloc(sizeof(double) * 3 * n, st));
  LW_CUDA_TRY(bn.alloc(sizeof(double) * 3 * n, st));
  LW_CUDA_TRY(bu.alloc(sizeof(double) * n, st));
  LW_CUDA_TRY(be.alloc(sizeof(long long) * n, st));
  LW_CUDA_TRY(bp.alloc(sizeof(double) * n, st));
  LW_CUDA_TRY(bo.alloc(sizeof(double) * n, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bx.p, x, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bn.p, nrm, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bu.p, u, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  k_light_sample_dbg<<<grid_for(n, 128, 1 << 30), 128, lt_smem_bytes(c), st>>>(c->S, bx.as<double>(), bn.as<double>(), bu.as<double>(),
                                                                 n, be.as<long long>(), bp.as<double>(), bo.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_e, be.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_psel, bp.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_u, bo.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_ctx_light_pdf(lw_ctx* c, const int64_t* e, const double* x, const double* nrm, int64_t n, double* out_psel) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  LW_CHECK_ARG(c->lt_nodes > 0, "the scene has no light hierarchy (pack_scene(..., lights='tree'))");
  if (n <= 0) return LW_OK;
  for (int64_t i = 0; i < n; i++) LW_CHECK_ARG(e[i] >= 0 && e[i] < c->S.nemit, "emitter index out of range");
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  DevBuf be, bx, bn, bp;
  LW_CUDA_TRY(be.alloc(sizeof(long long) * n, st));
  LW_CUDA_TRY(bx.alloc(sizeof(double) * 3 * n, st));
  LW_CUDA_TRY(bn.alloc(sizeof(double) * 3 * n, st));
  LW_CUDA_TRY(bp.alloc(sizeof(double) * n, st));
  LW_CUDA_TRY(cudaMemcpyAsync(be.p, e, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bx.p, x, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bn.p, nrm, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  k_light_pdf_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->S, be.as<long long>(), bx.as<double>(), bn.as<double>(),
                                                              n, bp.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_psel, bp.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_ctx_env_pyramid_info(lw_ctx* c, int32_t* nlevels) {
  LW_CHECK_ARG(c && c->has_scene && nlevels, "no scene");
  *nlevels = c->S.env_mode == LW_LIGHTS_ENV_PYRAMID ? c->S.env_pyr.nl : 0;
  return LW_OK;
}

int lw_ctx_env_sample(lw_ctx* c, const int64_t* pk, const double* uv, int64_t n, int64_t* out_t, double* out_p,
                      double* out_uv) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  LW_CHECK_ARG(c->S.env_mode == LW_LIGHTS_ENV_PYRAMID, "the scene has no environment pyramid (pack_scene(..., env_sampling='pyramid'))");
  if (n <= 0) return LW_OK;
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  DevBuf bk, bu, bt, bp, bo;
  LW_CUDA_TRY(bk.alloc(sizeof(long long) * n, st));
  LW_CUDA_TRY(bu.alloc(sizeof(double) * 2 * n, st));
  LW_CUDA_TRY(bt.alloc(sizeof(long long) * n, st));
  LW_CUDA_TRY(bp.alloc(sizeof(double) * n, st));
  LW_CUDA_TRY(bo.alloc(sizeof(double) * 2 * n, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bk.p, pk, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bu.p, uv, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, st));
  k_env_sample_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->S, bk.as<long long>(), bu.as<double>(), n,
                                                               bt.as<long long>(), bp.as<double>(), bo.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_t, bt.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_p, bp.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_uv, bo.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_ctx_env_pdf(lw_ctx* c, const int64_t* pk, const int64_t* tx, int64_t n, double* out_p) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  LW_CHECK_ARG(c->S.env_mode == LW_LIGHTS_ENV_PYRAMID, "the scene has no environment pyramid (pack_scene(..., env_sampling='pyramid'))");
  if (n <= 0) return LW_OK;
  int64_t nt = (int64_t)c->S.env_w * c->S.env_h;
  for (int64_t i = 0; i < n; i++) LW_CHECK_ARG(tx[i] >= 0 && tx[i] < nt, "texel index out of range");
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  DevBuf bk, bt, bp;
  LW_CUDA_TRY(bk.alloc(sizeof(long long) * n, st));
  LW_CUDA_TRY(bt.alloc(sizeof(long long) * n, st));
  LW_CUDA_TRY(bp.alloc(sizeof(double) * n, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bk.p, pk, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(bt.p, tx, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  k_env_pdf_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->S, bk.as<long long>(), bt.as<long long>(), n,
                                                            bp.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_p, bp.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_ctx_set_lpe(lw_ctx* c, int32_t nlayers, int32_t nstates, const int16_t* trans, const uint8_t* accept,
                   int32_t start) {
  LW_CHECK_ARG(c && c->configured, "lw_render_configure must precede lw_ctx_set_lpe");
  cudaSetDevice(c->device);
  LW_STATUS_TRY(pass_fold(c));
  c->epoch++;  // the layer tables are baked into the wave graph
  free_lpe(c);
  if (nlayers == 0) return LW_OK;
  LW_CHECK_ARG(nlayers > 0 && nlayers <= 8 && nstates > 0 && trans && accept && start >= 0 && start < nstates,
               "bad LPE tables");
  for (int64_t k = 0; k < (int64_t)nstates * LW_EV_COUNT; k++)
    LW_CHECK_ARG(trans[k] >= 0 && trans[k] < nstates, "LPE transition out of range");
  short* dt;
  unsigned char* da;
  unsigned long long* dfb;
  cudaStream_t st = c->stream;
  LW_CUDA_TRY(cudaMallocAsync((void**)&dt, sizeof(short) * nstates * LW_EV_COUNT, st));
  LW_CUDA_TRY(cudaMallocAsync((void**)&da, nstates, st));
  LW_CUDA_TRY(cudaMallocAsync((void**)&dfb, sizeof(unsigned long long) * 3 * c->fb_pixels * nlayers, st));
  LW_CUDA_TRY(cudaMemcpyAsync(dt, trans, sizeof(short) * nstates * LW_EV_COUNT, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemcpyAsync(da, accept, nstates, cudaMemcpyHostToDevice, st));
  LW_CUDA_TRY(cudaMemsetAsync(dfb, 0, sizeof(unsigned long long) * 3 * c->fb_pixels * nlayers, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  c->lpe = LwLpe{dt, da, start, nlayers, dfb, c->fb_pixels};
  return LW_OK;
}

int lw_ctx_lpe_download(lw_ctx* c, int32_t layer, int64_t* fb) {
  LW_CHECK_ARG(c && fb && layer >= 0 && layer < c->lpe.nlayers, "no such LPE layer");
  LW_CUDA_TRY(cudaMemcpyAsync(fb, c->lpe.fb + (size_t)layer * 3 * c->lpe.npix,
                              sizeof(int64_t) * 3 * c->lpe.npix, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_ctx_lpe_upload(lw_ctx* c, int32_t layer, const int64_t* fb) {
  LW_CHECK_ARG(c && fb && layer >= 0 && layer < c->lpe.nlayers, "no such LPE layer");
  LW_CUDA_TRY(cudaMemcpyAsync(c->lpe.fb + (size_t)layer * 3 * c->lpe.npix, fb, sizeof(int64_t) * 3 * c->lpe.npix,
                              cudaMemcpyHostToDevice, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

// ---- known-answer surface of the render math ----------------------------------------------------

}  // extern "C"

namespace {
struct DbgIO {  // device copies of host inputs / outputs of one debug call, on one stream
  cudaStream_t st;
  std::vector<DevBuf*> bufs;
  explicit DbgIO(cudaStream_t s) : st(s) {}
  ~DbgIO() {
    for (DevBuf* b : bufs) delete b;
  }
  template <class T>
  T* in(const void* host, size_t bytes) {
    DevBuf* b = new DevBuf();
    bufs.push_back(b);
    if (b->alloc(bytes, st) != cudaSuccess) return nullptr;
    if (cudaMemcpyAsync(b->p, host, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return nullptr;
    return (T*)b->p;
  }
  template <class T>
  T* out(size_t bytes) {
    DevBuf* b = new DevBuf();
    bufs.push_back(b);
    if (b->alloc(bytes, st) != cudaSuccess) return nullptr;
    return (T*)b->p;
  }
};
}  // namespace

extern "C" {

#define LW_DBG_PTR(p)                                \
  do {                                               \
    if (!(p)) {                                      \
      set_error("debug call: device buffer failed"); \
      return LW_ERR_NOMEM;                           \
    }                                                \
  } while (0)

int lw_bsdf_eval_batch(const lw_material* m, const double* wo, const double* wi, int64_t n, double* out_f,
                       double* out_pdf) {
  LW_CHECK_ARG(m && wo && wi && out_f && out_pdf && n >= 0, "bad arguments");
  LW_CHECK_ARG(m->nlayers >= 0 && m->nlayers <= LW_MAX_LAYERS, "bad material");
  if (n == 0) return LW_OK;
  cudaStream_t st = cudaStreamPerThread;
  DbgIO io(st);
  const double* a = io.in<double>(wo, sizeof(double) * 3 * n);
  const double* b = io.in<double>(wi, sizeof(double) * 3 * n);
  double* f = io.out<double>(sizeof(double) * 3 * n);
  double* p = io.out<double>(sizeof(double) * n);
  LW_DBG_PTR(a && b && f && p);
  k_bsdf_eval_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(*m, a, b, n, f, p);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_f, f, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_pdf, p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_bsdf_sample_batch(const lw_material* m, const double* wo, const int32_t* front, const double* uv, int64_t n,
                         double* out_wi, double* out_weight, double* out_pdf, int32_t* out_flags) {
  LW_CHECK_ARG(m && wo && front && uv && out_wi && out_weight && out_pdf && out_flags && n >= 0, "bad arguments");
  LW_CHECK_ARG(m->nlayers >= 0 && m->nlayers <= LW_MAX_LAYERS, "bad material");
  if (n == 0) return LW_OK;
  cudaStream_t st = cudaStreamPerThread;
  DbgIO io(st);
  const double* a = io.in<double>(wo, sizeof(double) * 3 * n);
  const int* fr = io.in<int>(front, sizeof(int32_t) * n);
  const double* u = io.in<double>(uv, sizeof(double) * 2 * n);
  double* wi = io.out<double>(sizeof(double) * 3 * n);
  double* w = io.out<double>(sizeof(double) * 3 * n);
  double* p = io.out<double>(sizeof(double) * n);
  int* fl = io.out<int>(sizeof(int32_t) * n);
  LW_DBG_PTR(a && fr && u && wi && w && p && fl);
  k_bsdf_sample_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(*m, a, fr, u, n, wi, w, p, fl);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_wi, wi, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_weight, w, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_pdf, p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaMemcpyAsync(out_flags, fl, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_mis_weight_batch(const double* pdf_a, const double* pdf_b, int64_t n, double* out) {
  LW_CHECK_ARG(pdf_a && pdf_b && out && n >= 0, "bad arguments");
  if (n == 0) return LW_OK;
  cudaStream_t st = cudaStreamPerThread;
  DbgIO io(st);
  const double* a = io.in<double>(pdf_a, sizeof(double) * n);
  const double* b = io.in<double>(pdf_b, sizeof(double) * n);
  double* o = io.out<double>(sizeof(double) * n);
  LW_DBG_PTR(a && b && o);
  k_mis_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(a, b, n, o);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out, o, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  LW_CUDA_TRY(cudaStreamSynchronize(st));
  return LW_OK;
}

int lw_ctx_nee_light_sample(lw_ctx* c, const double* p, const double* ngf, const double* uv, int64_t n, double* out_wi,
                            double* out_le, double* out_pdf, double* out_tmax, int64_t* out_emitter) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  LW_CHECK_ARG(p && ngf && uv && out_wi && out_le && out_pdf && out_tmax && out_emitter && n >= 0, "bad arguments");
  if (n == 0) return LW_OK;
  cudaSetDevice(c->device);
  DbgIO io(c->stream);
  const double* dp = io.in<double>(p, sizeof(double) * 3 * n);
  const double* dn = io.in<double>(ngf, sizeof(double) * 3 * n);
  const double* du = io.in<double>(uv, sizeof(double) * 2 * n);
  double* wi = io.out<double>(sizeof(double) * 3 * n);
  double* le = io.out<double>(sizeof(double) * 3 * n);
  double* pd = io.out<double>(sizeof(double) * n);
  double* tm = io.out<double>(sizeof(double) * n);
  long long* em = io.out<long long>(sizeof(int64_t) * n);
  LW_DBG_PTR(dp && dn && du && wi && le && pd && tm && em);
  k_nee_light_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, c->stream>>>(c->S, dp, dn, du, n, wi, le, pd, tm, em);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_wi, wi, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_le, le, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_pdf, pd, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_tmax, tm, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_emitter, em, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

int lw_ctx_emission_pdf(lw_ctx* c, const double* o, const double* d, const int32_t* nprev, int64_t n, double* out_le,
                        double* out_pdf, int64_t* out_emitter) {
  LW_CHECK_ARG(c && c->has_scene, "no scene");
  LW_CHECK_ARG(o && d && nprev && out_le && out_pdf && out_emitter && n >= 0, "bad arguments");
  if (n == 0) return LW_OK;
  cudaSetDevice(c->device);
  DbgIO io(c->stream);
  const double* dO = io.in<double>(o, sizeof(double) * 3 * n);
  const double* dD = io.in<double>(d, sizeof(double) * 3 * n);
  const int* dN = io.in<int>(nprev, sizeof(int32_t) * n);
  double* le = io.out<double>(sizeof(double) * 3 * n);
  double* pd = io.out<double>(sizeof(double) * n);
  long long* em = io.out<long long>(sizeof(int64_t) * n);
  LW_DBG_PTR(dO && dD && dN && le && pd && em);
  k_emission_pdf_dbg<<<grid_for(n, 128, 1 << 30), 128, 0, c->stream>>>(c->S, dO, dD, dN, n, le, pd, em);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out_le, le, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_pdf, pd, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaMemcpyAsync(out_emitter, em, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  LW_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LW_OK;
}

}  // extern "C"

// lw_sah.cu -- binned-SAH render BVH (host, deterministic).
//
// The render traversal needs a good tree, not the reference's arrays (those come from the GPU
// median builder, lw_bvh_build.cu).  The split rule is fully specified so that the CPU oracle
// (oracle/lw_oracle.c, written separately) builds the identical tree:
//   * per triangle: lo/hi = component-wise min/max of its three vertices, c = 0.5*(lo+hi);
//   * segments are split in FIFO (breadth-first) order; internal nodes are numbered in that order;
//   * 16 bins per axis over the centroid bounds, bin = (int)((c - cmin) * (16 / ext)) clamped to 15;
//     axes with ext <= 0 are skipped;
//   * candidate planes i = 0..14 with both sides non-empty, cost = A(L)*nL + A(R)*nR with
//     A(b) = 2*((dx*dy + dy*dz) + dz*dx); the first strict minimum over (axis, plane) wins;
//   * split if a plane exists and (n > 7 or A(B) + cost < n*A(B)); if n > 7 and no plane exists
//     (coincident centroids) the segment is halved in its current order;
//   * partition is stable (left = bin <= plane).
// Every FP operation is a plain IEEE double op (-ffp-contract=off), so both builds agree bit for bit.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "lw_common.cuh"
#include "lw_host.h"

namespace lw {

namespace {

constexpr int kBins = 16;
constexpr int kMaxLeaf = 7;

struct Box {
  double lo[3], hi[3];
};

inline void box_empty(Box& b) {
  for (int a = 0; a < 3; a++) {
    b.lo[a] = INFINITY;
    b.hi[a] = -INFINITY;
  }
}

inline void box_grow(Box& b, const double* lo, const double* hi) {
  for (int a = 0; a < 3; a++) {
    if (lo[a] < b.lo[a]) b.lo[a] = lo[a];
    if (hi[a] > b.hi[a]) b.hi[a] = hi[a];
  }
}

inline double box_area(const Box& b) {
  double dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return 2.0 * ((dx * dy + dy * dz) + dz * dx);
}

struct Seg {
  int64_t start, n;
  int64_t parent;  // internal node id, -1 = root
  int side;
};

inline int32_t leaf_ref32(int64_t start, int64_t count) { return (int32_t)(-(1 + ((start << 3) | count))); }

}  // namespace

int sah_build_host(const double* verts, int64_t n, SahBVH& out) {
  out.nodes.clear();
  out.order.assign(n, 0);
  out.root_ref = leaf_ref32(0, 0);
  for (int a = 0; a < 6; a++) out.root_box[a] = 0.0;
  if (n == 0) return LW_OK;
  if (n >= (1LL << 28)) {
    set_error("sah build: at most 2^28 triangles");
    return LW_ERR_INVALID;
  }
  std::vector<double> tlo(3 * n), thi(3 * n), cen(3 * n);
  for (int64_t i = 0; i < n; i++) {
    const double* v = verts + 9 * i;
    for (int a = 0; a < 3; a++) {
      double lo = v[a], hi = v[a];
      if (v[3 + a] < lo) lo = v[3 + a];
      if (v[6 + a] < lo) lo = v[6 + a];
      if (v[3 + a] > hi) hi = v[3 + a];
      if (v[6 + a] > hi) hi = v[6 + a];
      tlo[3 * i + a] = lo;
      thi[3 * i + a] = hi;
      cen[3 * i + a] = 0.5 * (lo + hi);
    }
    out.order[i] = i;
  }
  std::vector<int64_t>& ids = out.order;
  std::vector<int64_t> tmp(n);
  std::vector<Seg> fifo;
  fifo.reserve(2 * (n / 2 + 1));
  fifo.push_back({0, n, -1, 0});
  size_t head = 0;
  while (head < fifo.size()) {
    Seg sg = fifo[head++];
    const int64_t* sid = ids.data() + sg.start;
    Box B, Cb;
    box_empty(B);
    box_empty(Cb);
    for (int64_t k = 0; k < sg.n; k++) {
      int64_t t = sid[k];
      box_grow(B, &tlo[3 * t], &thi[3 * t]);
      box_grow(Cb, &cen[3 * t], &cen[3 * t]);
    }
    if (sg.parent < 0)
      for (int a = 0; a < 3; a++) {
        out.root_box[a] = B.lo[a];
        out.root_box[3 + a] = B.hi[a];
      }
    int best_axis = -1, best_plane = -1;
    double best_cost = INFINITY;
    Box best_l, best_r;
    int64_t best_nl = 0;
    if (sg.n > 1) {
      for (int a = 0; a < 3; a++) {
        double ext = Cb.hi[a] - Cb.lo[a];
        if (!(ext > 0.0)) continue;
        double scale = (double)kBins / ext;
        int64_t cnt[kBins];
        Box bb[kBins];
        for (int b = 0; b < kBins; b++) {
          cnt[b] = 0;
          box_empty(bb[b]);
        }
        for (int64_t k = 0; k < sg.n; k++) {
          int64_t t = sid[k];
          int b = (int)((cen[3 * t + a] - Cb.lo[a]) * scale);
          if (b > kBins - 1) b = kBins - 1;
          cnt[b]++;
          box_grow(bb[b], &tlo[3 * t], &thi[3 * t]);
        }
        Box rbox[kBins];
        int64_t rcnt[kBins];
        Box acc;
        box_empty(acc);
        int64_t ac = 0;
        for (int b = kBins - 1; b >= 1; b--) {
          box_grow(acc, bb[b].lo, bb[b].hi);
          ac += cnt[b];
          rbox[b] = acc;
          rcnt[b] = ac;
        }
        box_empty(acc);
        ac = 0;
        for (int p = 0; p < kBins - 1; p++) {
          box_grow(acc, bb[p].lo, bb[p].hi);
          ac += cnt[p];
          int64_t nr = rcnt[p + 1];
          if (ac == 0 || nr == 0) continue;
          double cost = box_area(acc) * (double)ac + box_area(rbox[p + 1]) * (double)nr;
          if (cost < best_cost) {
            best_cost = cost;
            best_axis = a;
            best_plane = p;
            best_l = acc;
            best_r = rbox[p + 1];
            best_nl = ac;
          }
        }
      }
    }
    bool split = false, halve = false;
    if (best_axis >= 0) {
      double aB = box_area(B);
      split = sg.n > kMaxLeaf || (aB + best_cost) < (double)sg.n * aB;
    } else if (sg.n > kMaxLeaf) {
      split = halve = true;
    }
    if (!split) {
      int32_t ref = leaf_ref32(sg.start, sg.n);
      if (sg.parent < 0)
        out.root_ref = ref;
      else
        out.nodes[sg.parent].ref[sg.side] = ref;
      continue;
    }
    int64_t id = (int64_t)out.nodes.size();
    out.nodes.emplace_back();
    SahNode& nd = out.nodes.back();
    memset(&nd, 0, sizeof(nd));
    if (sg.parent < 0)
      out.root_ref = (int32_t)id;
    else
      out.nodes[sg.parent].ref[sg.side] = (int32_t)id;
    int64_t nl;
    Box lb, rb;
    int64_t* w = ids.data() + sg.start;
    if (halve) {
      nl = sg.n / 2;
      box_empty(lb);
      box_empty(rb);
      for (int64_t k = 0; k < sg.n; k++) {
        int64_t t = w[k];
        box_grow(k < nl ? lb : rb, &tlo[3 * t], &thi[3 * t]);
      }
    } else {
      nl = best_nl;
      lb = best_l;
      rb = best_r;
      double scale = (double)kBins / (Cb.hi[best_axis] - Cb.lo[best_axis]);
      int64_t li = 0, ri = 0;
      for (int64_t k = 0; k < sg.n; k++) {
        int64_t t = w[k];
        int b = (int)((cen[3 * t + best_axis] - Cb.lo[best_axis]) * scale);
        if (b > kBins - 1) b = kBins - 1;
        if (b <= best_plane)
          w[li++] = t;
        else
          tmp[ri++] = t;
      }
      memcpy(w + li, tmp.data(), sizeof(int64_t) * ri);
    }
    SahNode& nn = out.nodes[id];
    for (int a = 0; a < 3; a++) {
      nn.box[a] = lb.lo[a];
      nn.box[3 + a] = lb.hi[a];
      nn.box[6 + a] = rb.lo[a];
      nn.box[9 + a] = rb.hi[a];
    }
    fifo.push_back({sg.start, nl, id, 0});
    fifo.push_back({sg.start + nl, sg.n - nl, id, 1});
  }
  return LW_OK;
}

}  // namespace lw

// gs_audit.cuh -- device-side packer auditor.
//
// The reference audits a node's geometry with check_node (packer.py:327-388):
// placements pairwise disjoint, free rectangles disjoint from placements, no
// free rectangle contained in another (exact duplicates: the later one is the
// breach), and coverage -- free ∪ placed must tile the plane exactly -- by
// painting both onto an integer raster (skipped when it would need more than
// 20x resolution).  Here every coordinate is already an exact integer on the
// compiler's scaled grid, so coverage is decided exactly on the grid
// *compressed* to the rectangles' own edges: each compressed cell is either
// inside or outside every rectangle, so "neither free nor placed" (gap) and
// "both" (overlap) are cell-level facts, at any scale.
//
// One warp per (run, node); breach bits are OR-ed per run.
#pragma once
#include "gs_kernel.cuh"

namespace gs {

enum : unsigned {
  AUD_PLACED_OVERLAP = 1u,     // two placements intersect
  AUD_FREE_PLACED = 2u,        // a free rect intersects a placement
  AUD_FREE_CONTAINED = 4u,     // a free rect is contained in another
  AUD_GAP = 8u,                // plane area neither free nor placed
  AUD_DOUBLE = 16u,            // plane area both free and placed
  AUD_TOO_BIG = 32u,           // node exceeds the auditor's scratch (not audited)
};

constexpr int AUD_MAX_RECTS = 256;   // free + placed rectangles per node

// Audit one node: `rects[0..nf)` free, `rects[nf..nf+np)` placed.  `xs`/`ys`
// (and xs2/ys2) are warp scratch of 2*(nf+np)+2 ints.  Returns the breach
// bits (all lanes).
__device__ unsigned audit_node(const int4* rects, int nf, int np, int side_x, int side_y,
                               int* xs, int* ys, int* xs2, int* ys2, int lane) {
  const int n = nf + np;
  unsigned bad = 0u;
  // pairwise checks: pair index t -> (i, j), i < j
  const long long pairs = (long long)n * (n - 1) / 2;
  for (long long t = lane; t < pairs; t += 32) {
    // invert t = j*(j-1)/2 + i
    int j = (int)((1.0 + sqrt(1.0 + 8.0 * (double)t)) / 2.0);
    while ((long long)j * (j - 1) / 2 > t) j--;
    while ((long long)(j + 1) * j / 2 <= t) j++;
    const int i = (int)(t - (long long)j * (j - 1) / 2);
    const int4 a = rects[i], b = rects[j];
    const bool inter = r_intersects(a, b);
    if (i >= nf) {                          // both placed
      if (inter) bad |= AUD_PLACED_OVERLAP;
    } else if (j >= nf) {                   // free i, placed j
      if (inter) bad |= AUD_FREE_PLACED;
    } else {                                // both free (i < j)
      // i contained in j is a breach; j contained in i is a breach unless
      // they are equal (then only the later one, j, counts: packer.py:352-355)
      if (r_contains(b, a) && !r_eq(a, b)) bad |= AUD_FREE_CONTAINED;
      if (r_contains(a, b)) bad |= AUD_FREE_CONTAINED;
    }
  }
  // compressed coordinates: plane edges + every rectangle edge
  const int m = 2 * n + 2;
  for (int k = lane; k < m; k += 32) {
    if (k == 0) { xs[k] = 0; ys[k] = 0; }
    else if (k == 1) { xs[k] = side_x; ys[k] = side_y; }
    else {
      const int4 r = rects[(k - 2) >> 1];
      const bool hi = (k - 2) & 1;
      xs[k] = hi ? r.x + r.z : r.x;
      ys[k] = hi ? r.y + r.w : r.y;
    }
  }
  __syncwarp();
  // sort both coordinate lists into xs2/ys2 (rank counting; ties by index)
  for (int k = lane; k < m; k += 32) {
    const int x = xs[k], y = ys[k];
    int rx = 0, ry = 0;
    for (int l = 0; l < m; l++) {
      rx += xs[l] < x || (xs[l] == x && l < k);
      ry += ys[l] < y || (ys[l] == y && l < k);
    }
    xs2[rx] = x;
    ys2[ry] = y;
  }
  __syncwarp();
  xs = xs2;
  ys = ys2;
  // cells [xs[a], xs[a+1]) x [ys[b], ys[b+1]) of positive area inside the plane
  const int cells = (m - 1) * (m - 1);
  for (int c = lane; c < cells; c += 32) {
    const int a = c % (m - 1), b = c / (m - 1);
    const int x0 = xs[a], x1 = xs[a + 1], y0 = ys[b], y1 = ys[b + 1];
    if (x0 == x1 || y0 == y1 || x1 > side_x || y1 > side_y || x0 < 0 || y0 < 0) continue;
    bool in_free = false, in_placed = false;
    for (int k = 0; k < n; k++) {
      const int4 r = rects[k];
      const bool in = r.x <= x0 && x1 <= r.x + r.z && r.y <= y0 && y1 <= r.y + r.w;
      if (in) { if (k < nf) in_free = true; else in_placed = true; }
    }
    if (!in_free && !in_placed) bad |= AUD_GAP;
    if (in_free && in_placed) bad |= AUD_DOUBLE;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad |= __shfl_xor_sync(FULL, bad, o);
  return bad;
}

struct AuditArgs {
  // geometry mode (standalone): per node nf free + np placed rects at
  // rects[node * cap ...]; session mode: read from the run arenas
  const int4* rects; const int* nfree; const int* nplaced; int cap;
  int n_nodes; int side_x, side_y;
  // session mode
  const gs_batch_t* in; const char* arena; const long long* ws_off; int n_runs;
  int4* scratch;            // per warp: AUD_MAX_RECTS rects (session mode)
  unsigned* out;            // per node (geometry) or per run (session)
};

__global__ void __launch_bounds__(128) gs_audit_geometry_kernel(AuditArgs a) {
  __shared__ int xs[4][2 * AUD_MAX_RECTS + 2], ys[4][2 * AUD_MAX_RECTS + 2];
  __shared__ int xs2[4][2 * AUD_MAX_RECTS + 2], ys2[4][2 * AUD_MAX_RECTS + 2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int node = blockIdx.x * 4 + wib;
  if (node >= a.n_nodes) return;
  const int nf = a.nfree[node], np = a.nplaced[node];
  unsigned bad;
  if (nf + np > AUD_MAX_RECTS || nf + np > a.cap) bad = AUD_TOO_BIG;
  else bad = audit_node(a.rects + (size_t)node * a.cap, nf, np, a.side_x, a.side_y,
                        xs[wib], ys[wib], xs2[wib], ys2[wib], lane);
  if (lane == 0) a.out[node] = bad;
}

__global__ void __launch_bounds__(128) gs_audit_session_kernel(AuditArgs a) {
  __shared__ int xs[4][2 * AUD_MAX_RECTS + 2], ys[4][2 * AUD_MAX_RECTS + 2];
  __shared__ int xs2[4][2 * AUD_MAX_RECTS + 2], ys2[4][2 * AUD_MAX_RECTS + 2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int run = blockIdx.x * 4 + wib;
  if (run >= a.n_runs) return;
  const gs_scenario_t& sc = a.in->runs[run];
  const gs_function_t* fs = &a.in->funcs[sc.func_off];
  long long ring = 0;
  for (int f = 0; f < sc.n_funcs; f++) if (fs[f].max_queue > 0) ring += fs[f].max_queue;
  const Layout L = gs_make_layout(sc.n_nodes, sc.n_funcs, sc.cap_pods, sc.cap_rects,
                                  sc.cap_returned, ring);
  const char* base = a.arena + a.ws_off[run];
  const int4* rect = reinterpret_cast<const int4*>(base + L.n_rect);
  const int* nfree = reinterpret_cast<const int*>(base + L.n_nfree);
  const int* flags = reinterpret_cast<const int*>(base + L.p_flags);
  const int* node_of = reinterpret_cast<const int*>(base + L.p_node);
  const int* px = reinterpret_cast<const int*>(base + L.p_x);
  const int* py = reinterpret_cast<const int*>(base + L.p_y);
  const int* pw = reinterpret_cast<const int*>(base + L.p_w);
  const int* ph = reinterpret_cast<const int*>(base + L.p_h);
  int4* list = a.scratch + (size_t)(blockIdx.x * 4 + wib) * AUD_MAX_RECTS;
  unsigned bad = 0u;
  for (int g = 0; g < sc.n_nodes; g++) {
    const int nf = nfree[g];
    if (nf > AUD_MAX_RECTS) { bad |= AUD_TOO_BIG; continue; }
    for (int j = lane; j < nf; j += 32) list[j] = rect[(size_t)g * sc.cap_rects + j];
    int np = 0;
    for (int s0 = 0; s0 < sc.cap_pods; s0 += 32) {
      const int slot = s0 + lane;
      const bool take = slot < sc.cap_pods && (flags[slot] & PF_PLACED) && node_of[slot] == g;
      const unsigned bal = __ballot_sync(FULL, take);
      const int k = nf + np + __popc(bal & ((1u << lane) - 1u));
      if (take && k < AUD_MAX_RECTS) list[k] = make_int4(px[slot], py[slot], pw[slot], ph[slot]);
      np += __popc(bal);
    }
    __syncwarp();
    if (nf + np > AUD_MAX_RECTS) { bad |= AUD_TOO_BIG; continue; }
    bad |= audit_node(list, nf, np, sc.side_x, sc.side_y, xs[wib], ys[wib], xs2[wib], ys2[wib], lane);
    __syncwarp();
  }
  if (lane == 0) a.out[run] = bad;
}

}  // namespace gs

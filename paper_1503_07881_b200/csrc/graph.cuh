// graph.cuh — the device-resident CSR pair owned by a gt_graph handle.
//
// Layout in HBM (all buffers owned by the handle, freed by gt_graph_free):
//   ids     int64 [N]     distinct node ids, ascending (convert.py:51-52)
//   out_off int64 [N+1]   exclusive prefix of out-degrees (convert.py:154-156)
//   out_adj int32 [E]     dense dst index per edge, ascending within a row
//   in_off  int64 [N+1]   exclusive prefix of in-degrees (convert.py:155-157)
//   in_adj  int32 [E]     dense src index per edge, ascending within a row
// The reference's per-node pools hold original int64 ids (convert.py:159-164);
// gt_graph_export gathers ids[adj] to reproduce them exactly.
#pragma once

#include "common.cuh"

struct gt_graph {
  int64_t n = 0;
  int64_t e = 0;
  int kbits = 1;  // bits of a dense index inside packed keys
  int64_t* ids = nullptr;
  int64_t* out_off = nullptr;
  int32_t* out_adj = nullptr;
  int64_t* in_off = nullptr;
  int32_t* in_adj = nullptr;
  // undirected simple-edge count m, set by the first triangle count (-1 before)
  mutable int64_t m_und = -1;
};

namespace gt {
// Undirected degree |out(i) ∪ in(i) \ {i}| of every node (graphs.py:163-167)
// into deg[N], cat[N+1] = out_off + in_off (offsets of the concatenated
// out(i) ++ in(i) candidate slots) and one keep bit per slot (a slot is an
// undirected neighbour unless it is a self-loop or an in-slot whose source is
// also in the out-row): returned, valid until the next call that uses the
// WS_RANKMAP workspace slot (triangles.cu).
uint32_t* undirected_degrees(const gt_graph* g, int64_t* cat, int32_t* deg, const char* phase);

inline int bits_for(int64_t n) {  // bits needed to hold values 0..n-1 (>= 1)
  int b = 1;
  while (b < 63 && (int64_t(1) << b) < n) ++b;
  return b;
}
}  // namespace gt

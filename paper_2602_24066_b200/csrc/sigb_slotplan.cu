// Level-slot planner (sigb_slot.cuh): assigns every closure node to one thread
// of a one-path CTA, lays out the shared-memory partial tables and the
// letter-major gradient parking buffer.  Host code, once per word set.
#include <algorithm>

#include "sigb_internal.h"
#include "sigb_slot.cuh"

namespace sigb {

bool plan_slots(const Trie& t, SlotHost& out, std::string& why) {
  using namespace slot;
  const int64_t Wc = (int64_t)t.code.size();
  const int N = t.max_len;
  const int d = (int)t.d;
  if (N < 1 || N > 7 || d > 254) {
    why = "level-slot kernels need depth <= 7 and d <= 254";
    return false;
  }
  std::vector<int64_t> lstart(N + 2, Wc);
  for (int64_t i = Wc - 1; i >= 0; --i) lstart[t.len[i]] = i;
  lstart[N + 1] = Wc;
  for (int l = N; l >= 1; --l)
    if (lstart[l] > lstart[l + 1]) lstart[l] = lstart[l + 1];
  std::vector<int> n(N + 2, 0), tcount(N + 2, 0), tstart(N + 2, 0);
  int TPB = 0;
  for (int l = 1; l <= N; ++l) {
    n[l] = (int)(lstart[l + 1] - lstart[l]);
    const int need = (n[l] + KS - 1) / KS;
    tcount[l] = (need + 31) / 32 * 32;
    tstart[l] = TPB;
    TPB += tcount[l];
  }
  if (TPB > 512 || TPB == 0) {
    why = "closure too large for one level-slot CTA";
    return false;
  }
  out = SlotHost();
  out.N = N;
  out.TPB = TPB;
  // -- shared-memory layout (elements) -------------------------------------------
  auto al4 = [](int x) { return (x + 3) / 4 * 4; };
  int o = 8;  // ONES
  out.a_off = o;
  o += kChunkS * d * AW;
  out.t_off = o = al4(o);
  out.lvl.assign(2 * N + 4, 0);
  // each level's T-vectors are followed by 8 pad elements: the kernels read a
  // parent's T-vector as 8 values (ld8) and use only the first nT, so the
  // over-read must not touch the next level while it is being written
  for (int l = 1; l <= N; ++l) {
    out.lvl[l] = o;
    o += n[l] * t_stride(N, l) + 8;
  }
  out.t_size = o - out.t_off;
  // parking: letter-major blocks padded to float4
  std::vector<int> cntz(d, 0);
  for (int64_t i = 0; i < Wc; ++i) cntz[t.code[i] % (uint64_t)d]++;
  std::vector<int> base(d + 1, 0);
  for (int z = 0; z < d; ++z) base[z + 1] = base[z] + al4(cntz[z]);
  out.red_off.assign(d + 1, 0);
  for (int z = 0; z <= d; ++z) out.red_off[z] = base[z] / 4;
  out.pstride = base[d];
  out.park_off = o = al4(o);
  o += std::max(kRedS * out.pstride, (kChunkS + 1) * d) + 8;
  out.fwd_smem = o;
  out.tm_off = o = al4(o);
  o += out.t_size;
  o = al4(o);
  for (int l = 1; l <= N; ++l) {
    out.lvl[N + 2 + l] = o;
    o += n[l] * p_stride(N, l) + 8;
  }
  out.p_off = out.lvl[N + 3];
  out.p_size = o - out.p_off;
  out.bwd_smem = o + 8;
  if (out.bwd_smem >= 65535) {
    why = "level-slot tables exceed 16-bit shared-memory offsets";
    return false;
  }
  // -- per-thread slots ----------------------------------------------------------
  out.tinfo.assign(TPB, 0);
  out.meta0.assign((size_t)KS * TPB, 0);
  out.meta1.assign((size_t)KS * TPB, 0);
  out.pos.assign((size_t)KS * TPB, 0xFFFF);
  out.cidx.assign((size_t)KS * TPB, -1);
  out.eidx.assign((size_t)KS * TPB, -1);
  std::vector<int> fill(base.begin(), base.end() - 1);
  for (int l = 1; l <= N; ++l) {
    for (int i = 0; i < tcount[l]; ++i) {
      const int tid = tstart[l] + i;
      const int lo = (int)((int64_t)i * n[l] / tcount[l]), hi = (int)((int64_t)(i + 1) * n[l] / tcount[l]);
      const int cnt = hi - lo;
      out.tinfo[tid] = l | (cnt << 4) | (lo << 8);
      for (int k = 0; k < cnt; ++k) {
        const int64_t u = lstart[l] + lo + k;
        const int letter = (int)(t.code[u] % (uint64_t)d);
        const int nT = t.md[u] - l + 1;
        int pT = 0;
        if (l > 1) pT = out.lvl[l - 1] + (int)(t.parent[u] - lstart[l - 1]) * t_stride(N, l - 1);
        out.meta0[(size_t)k * TPB + tid] = (unsigned)pT | ((unsigned)letter << 16) | ((unsigned)nT << 24);
        const int cf = t.child_count[u] ? (int)(t.child_first[u] - lstart[l + 1]) : 0;
        out.meta1[(size_t)k * TPB + tid] = (unsigned)cf | ((unsigned)t.child_count[u] << 16);
        out.pos[(size_t)k * TPB + tid] = (unsigned short)fill[letter]++;
        out.cidx[(size_t)k * TPB + tid] = (int)u;
        out.eidx[(size_t)k * TPB + tid] = (int)t.emit[u];
      }
    }
  }
  return true;
}

}  // namespace sigb

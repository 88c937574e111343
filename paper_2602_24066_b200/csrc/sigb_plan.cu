// Execution plan of a word set: prefix closure, device tables, trie schedule.
//
// The reference kernels treat every (path, word) as an independent unit that
// replays all |w| prefixes of its word every step (_kernels.py:46-58).  Here
// the closure cl(I) is laid out once as a trie and cut into independent
// PARTS: a part is a run of consecutive sibling subtrees plus the chain of
// their common ancestors.  Chen's update of a word needs only its own
// prefixes, so parts never communicate in the forward;
// chain ancestors are recomputed redundantly by every part that needs them
// and emitted only by their owner part.  In the backward the adjoints of a
// replicated ancestor are kept as per-part partial sums, which is exact
// because the adjoint recursion is linear in them.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "sigb_internal.h"

namespace sigb {
namespace {

// Shared-memory budget a part's backward may use, in bytes, at 8-byte elements.
constexpr int64_t kPartSmemBudget = 200 * 1024;

int64_t node_cost(int level, int md) { return 3 + (md - level) + (md - level + 1); }

struct PartSpec {
  std::vector<int64_t> chain;  // ancestors, depth 1..k-1
  int64_t first_root, num_roots;
};

void split(const Trie& t, const std::vector<int64_t>& chain, int64_t first, int64_t count,
           int64_t budget, std::vector<PartSpec>& out) {
  int64_t chain_cost = 0;
  int chain_md = 0;
  for (int64_t r = first; r < first + count; ++r) chain_md = std::max(chain_md, t.md[r]);
  for (int64_t a : chain) chain_cost += node_cost((int)t.len[a], chain_md);
  int64_t r = first;
  while (r < first + count) {
    if (chain_cost + t.cost[r] > budget && t.child_count[r] > 0) {
      std::vector<int64_t> sub = chain;
      sub.push_back(r);
      split(t, sub, t.child_first[r], t.child_count[r], budget, out);
      ++r;
      continue;
    }
    int64_t acc = chain_cost + t.cost[r], e = r + 1;
    while (e < first + count && acc + t.cost[e] <= budget) acc += t.cost[e++];
    out.push_back(PartSpec{chain, r, e - r});
    r = e;
  }
}

}  // namespace
}  // namespace sigb

using namespace sigb;

// Builds the prefix closure cl(I) as a trie.  The parent of w is
// prefix_table[w, |w|-1]: taken from the DEVICE table builder
// (sigb_wordset_tables) when `stream_or_null` is a live stream, else by the
// same binary search on the host (sigb_fragment_plan_info, no GPU needed).
static int build_trie(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d, bool on_device,
                      cudaStream_t stream, Trie& t) {
  if (W < 1) return fail(SIGB_ERR_DOMAIN, "word set has no words to compute");
  if (d < 1) return fail(SIGB_ERR_DOMAIN, "alphabet size must be >= 1, got " + std::to_string(d));
  if (d > 255) return fail(SIGB_ERR_UNSUPPORTED, "the device kernels support d <= 255 letters");
  int64_t max_len = 0;
  for (int64_t i = 0; i < W; ++i) {
    if (lengths[i] < 1) return fail(SIGB_ERR_DOMAIN, "word sets may not contain the empty word");
    if (i > 0 && !(lengths[i] > lengths[i - 1] || (lengths[i] == lengths[i - 1] && codes[i] > codes[i - 1])))
      return fail(SIGB_ERR_DOMAIN, "words must be in canonical (length, code) order without duplicates");
    max_len = std::max(max_len, lengths[i]);
  }
  if (max_len > kMaxLevel)
    return fail(SIGB_ERR_UNSUPPORTED, "the device kernels support words of length <= " +
                                          std::to_string(kMaxLevel) + ", got " + std::to_string(max_len));
  // -- prefix closure cl(I) (wordsets.py:8-9, :441-443) -------------------------
  std::vector<uint64_t> pw(max_len + 1, 1);
  for (int k = 1; k <= max_len; ++k) pw[k] = pw[k - 1] * (uint64_t)d;  // d^max_len <= 2^64 (may wrap at the top)
  std::vector<std::pair<int64_t, uint64_t>> cl;
  cl.reserve((size_t)W * 2);
  for (int64_t i = 0; i < W; ++i)
    for (int64_t k = 1; k <= lengths[i]; ++k)
      cl.emplace_back(k, k == lengths[i] ? codes[i] : codes[i] / pw[lengths[i] - k]);
  std::sort(cl.begin(), cl.end());
  cl.erase(std::unique(cl.begin(), cl.end()), cl.end());
  t = Trie();
  t.d = d;
  t.max_len = (int)max_len;
  const int64_t Wc = (int64_t)cl.size();
  t.code.resize(Wc);
  t.len.resize(Wc);
  for (int64_t i = 0; i < Wc; ++i) { t.len[i] = cl[i].first; t.code[i] = cl[i].second; }
  t.emit.assign(Wc, -1);
  {
    int64_t j = 0;
    for (int64_t i = 0; i < W; ++i) {
      while (t.len[j] != lengths[i] || t.code[j] != codes[i]) ++j;
      t.emit[j] = i;
    }
  }
  t.parent.resize(Wc);
  if (on_device) {
    std::vector<int64_t> prefix((size_t)Wc * (max_len + 1));
    uint64_t* dc = nullptr;
    int64_t *dl = nullptr, *dp = nullptr, *ds = nullptr;
    SIGB_CUDA_TRY(cudaMalloc(&dc, sizeof(uint64_t) * Wc));
    SIGB_CUDA_TRY(cudaMalloc(&dl, sizeof(int64_t) * Wc));
    SIGB_CUDA_TRY(cudaMalloc(&dp, sizeof(int64_t) * Wc * (max_len + 1)));
    SIGB_CUDA_TRY(cudaMalloc(&ds, sizeof(int64_t) * (max_len + 2)));
    SIGB_CUDA_TRY(cudaMemcpyAsync(dc, t.code.data(), sizeof(uint64_t) * Wc, cudaMemcpyHostToDevice, stream));
    SIGB_CUDA_TRY(cudaMemcpyAsync(dl, t.len.data(), sizeof(int64_t) * Wc, cudaMemcpyHostToDevice, stream));
    int rc = launch_wordset_tables(dc, dl, Wc, d, max_len, nullptr, dp, nullptr, ds, nullptr, stream);
    if (rc != SIGB_OK) return rc;
    SIGB_CUDA_TRY(cudaMemcpyAsync(prefix.data(), dp, sizeof(int64_t) * prefix.size(), cudaMemcpyDeviceToHost,
                                  stream));
    SIGB_CUDA_TRY(cudaStreamSynchronize(stream));
    cudaFree(dc); cudaFree(dl); cudaFree(dp); cudaFree(ds);
    for (int64_t i = 0; i < Wc; ++i) t.parent[i] = t.len[i] == 1 ? -1 : prefix[(size_t)i * (max_len + 1) + t.len[i] - 1];
  } else {
    for (int64_t i = 0; i < Wc; ++i) {
      if (t.len[i] == 1) { t.parent[i] = -1; continue; }
      const std::pair<int64_t, uint64_t> key(t.len[i] - 1, t.code[i] / (uint64_t)d);
      auto it = std::lower_bound(cl.begin(), cl.end(), key);
      t.parent[i] = (it != cl.end() && *it == key) ? (int64_t)(it - cl.begin()) : -2;
    }
  }
  t.child_first.assign(Wc, 0);
  t.child_count.assign(Wc, 0);
  for (int64_t i = 0; i < Wc; ++i)
    if (t.len[i] > 1 && t.parent[i] < 0) return fail(SIGB_ERR_CUDA, "closure lost a prefix (table build failed)");
  for (int64_t i = Wc - 1; i >= 0; --i) {
    int64_t p = t.parent[i];
    if (p >= 0) { t.child_first[p] = i; t.child_count[p] += 1; }
  }
  t.md.resize(Wc);
  t.cost.resize(Wc);
  for (int64_t i = Wc - 1; i >= 0; --i) {
    int m = (int)t.len[i];
    for (int64_t c = t.child_first[i]; c < t.child_first[i] + t.child_count[i]; ++c) m = std::max(m, t.md[c]);
    t.md[i] = m;
  }
  for (int64_t i = Wc - 1; i >= 0; --i) {
    int64_t c = node_cost((int)t.len[i], t.md[i]);
    for (int64_t k = t.child_first[i]; k < t.child_first[i] + t.child_count[i]; ++k) c += t.cost[k];
    t.cost[i] = c;
  }
  return SIGB_OK;
}

extern "C" int sigb_fragment_plan_info(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d,
                                       int64_t* info) {
  if (!info) return fail(SIGB_ERR_DOMAIN, "info output pointer is NULL");
  Trie t;
  int rc = build_trie(codes, lengths, W, d, false, nullptr, t);
  if (rc) return rc;
  FragHost fh;
  std::string why;
  if (!plan_fragments(t, fh, why)) return fail(SIGB_ERR_UNSUPPORTED, why);
  info[0] = fh.NC; info[1] = fh.G; info[2] = fh.K; info[3] = fh.F; info[4] = fh.cpp;
  info[5] = (int64_t)t.code.size(); info[6] = (int64_t)fh.cost; info[7] = frag::supported(fh.NC, fh.G, fh.K);
  return SIGB_OK;
}

extern "C" int sigb_jit_source(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d, int dtype,
                               int backward, char* buf, size_t cap, size_t* len) {
  Trie t;
  int rc = build_trie(codes, lengths, W, d, false, nullptr, t);
  if (rc) return rc;
  if (!jit::eligible(t)) return fail(SIGB_ERR_UNSUPPORTED, "word set too large for generated kernels");
  JitHost h;
  jit::make_plan(t, h);
  const std::string src = jit::source(t, h, dtype, backward != 0);
  if (len) *len = src.size();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, src.size());
    std::memcpy(buf, src.data(), n);
    buf[n] = 0;
  }
  return SIGB_OK;
}

extern "C" int sigb_jit_precompile(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d, int dtype,
                                   int backward) {
  if (dtype != SIGB_F32 && dtype != SIGB_F64) return fail(SIGB_ERR_SHAPE, "unsupported dtype; use float64 or float32");
  Trie t;
  int rc = build_trie(codes, lengths, W, d, false, nullptr, t);
  if (rc) return rc;
  if (!jit::eligible(t)) return fail(SIGB_ERR_UNSUPPORTED, "word set too large for generated kernels");
  return jit::precompile(t, dtype, backward != 0);
}

extern "C" int sigb_plan_create(const uint64_t* codes, const int64_t* lengths, int64_t W, int64_t d,
                                sigb_plan** plan_out, void* stream_) {
  if (!plan_out) return fail(SIGB_ERR_DOMAIN, "plan output pointer is NULL");
  *plan_out = nullptr;
  cudaStream_t stream = (cudaStream_t)stream_;
  Trie t;
  {
    int rc = build_trie(codes, lengths, W, d, true, stream, t);
    if (rc) return rc;
  }
  const int64_t Wc = (int64_t)t.code.size();
  const int64_t max_len = t.max_len;
  // -- partition into parts -----------------------------------------------------
  const int64_t fixed = (int64_t)(kChunk + 1) * d + (int64_t)kChunk * max_len * d + 64;
  const int64_t budget = std::max<int64_t>(kPartSmemBudget / 8 - fixed, 64);
  int64_t n_roots = 0;
  while (n_roots < Wc && t.len[n_roots] == 1) ++n_roots;
  std::vector<PartSpec> specs;
  split(t, {}, 0, n_roots, budget, specs);

  sigb_plan* plan = new sigb_plan();
  cudaGetDevice(&plan->device);
  plan->d = d;
  plan->W = W;
  plan->Wc = Wc;
  plan->max_len = (int)max_len;
  plan->prefix_closed = (Wc == W);
  {
    bool full = plan->prefix_closed;
    std::vector<int64_t> cnt(max_len + 1, 0);
    for (int64_t i = 0; i < Wc; ++i) cnt[t.len[i]]++;
    uint64_t p = 1;
    for (int64_t n = 1; n <= max_len && full; ++n) {
      p *= (uint64_t)d;
      full = full && (uint64_t)cnt[n] == p;
    }
    plan->trunc_depth = full ? (int)max_len : 0;
  }
  plan->num_parts = (int)specs.size();
  std::vector<int4> nodeA, nodeB;
  std::vector<int> perm, lseg;
  std::vector<char> owned(Wc, 0);
  int64_t step_fmas = 0;
  for (const PartSpec& ps : specs) {
    // local nodes: chain + all subtree nodes of the roots, sorted (= canonical order)
    std::vector<int64_t> nodes(ps.chain.begin(), ps.chain.end());
    std::vector<int64_t> stack;
    for (int64_t r = ps.first_root; r < ps.first_root + ps.num_roots; ++r) stack.push_back(r);
    while (!stack.empty()) {
      int64_t v = stack.back();
      stack.pop_back();
      nodes.push_back(v);
      for (int64_t c = t.child_first[v]; c < t.child_first[v] + t.child_count[v]; ++c) stack.push_back(c);
    }
    std::sort(nodes.begin(), nodes.end());
    const int n = (int)nodes.size();
    auto local = [&](int64_t g) -> int {
      auto it = std::lower_bound(nodes.begin(), nodes.end(), g);
      return (it != nodes.end() && *it == g) ? (int)(it - nodes.begin()) : -1;
    };
    int roots_md = 0;
    for (int64_t r = ps.first_root; r < ps.first_root + ps.num_roots; ++r) roots_md = std::max(roots_md, t.md[r]);
    PartDesc pd;
    std::memset(&pd, 0, sizeof(pd));
    pd.n = n;
    pd.node_off = (int)nodeA.size();
    pd.lseg_off = (int)lseg.size();
    std::vector<int> mdl(n), lvl(n), toff(n, -1), tboff(n);
    const size_t chain_len = ps.chain.size();
    int tv = 0, tb = 0, depth = 0;
    for (int i = 0; i < n; ++i) {
      int64_t g = nodes[i];
      lvl[i] = (int)t.len[g];
      mdl[i] = (i < (int)chain_len) ? roots_md : t.md[g];
      depth = std::max(depth, lvl[i]);
      if (mdl[i] > lvl[i]) { toff[i] = tv; tv += mdl[i] - lvl[i]; }
      tboff[i] = tb;
      tb += mdl[i] - lvl[i] + 1;
    }
    pd.tv_size = tv;
    pd.tb_size = tb;
    pd.depth = depth;
    step_fmas += tb;
    for (int l = 0; l <= kMaxLevel + 1; ++l) pd.lvl[l] = n;
    for (int i = n - 1; i >= 0; --i) pd.lvl[lvl[i]] = i;
    for (int l = depth; l >= 1; --l)
      if (pd.lvl[l] == n && l < depth) pd.lvl[l] = pd.lvl[l + 1];
    pd.lvl[depth + 1] = n;
    for (int i = 0; i < n; ++i) {
      int64_t g = nodes[i];
      int owner;
      if (i < (int)chain_len) {
        owner = owned[g] ? 0 : 1;
        owned[g] = 1;
      } else {
        owner = 1;
        owned[g] = 1;
      }
      int ptoff = -1;
      if (t.parent[g] >= 0) {
        int pl = local(t.parent[g]);
        if (pl < 0) { delete plan; return fail(SIGB_ERR_CUDA, "internal: parent outside part"); }
        ptoff = toff[pl];
      }
      int letter = (int)(t.code[g] % (uint64_t)d);
      int cf = 0, cc = 0;
      if (i + 1 < (int)chain_len) {
        cf = i + 1; cc = 1;
      } else if (i + 1 == (int)chain_len) {
        cf = local(ps.first_root); cc = (int)ps.num_roots;
      } else if (t.child_count[g] > 0) {
        cf = local(t.child_first[g]); cc = (int)t.child_count[g];
      }
      nodeA.push_back(make_int4(ptoff, letter | (lvl[i] << 8) | (mdl[i] << 16) | (owner << 24), toff[i], tboff[i]));
      nodeB.push_back(make_int4((int)g, (int)t.emit[g], cf, cc));
    }
    // letter-sorted permutation for the per-letter gradient reduction
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return (nodeA[pd.node_off + a].y & 255) < (nodeA[pd.node_off + b].y & 255);
    });
    for (int i = 0; i < n; ++i) perm.push_back(order[i]);
    int pos = 0;
    for (int z = 0; z <= d; ++z) {
      while (pos < n && (nodeA[pd.node_off + order[pos]].y & 255) < z) ++pos;
      lseg.push_back(pos);
    }
    plan->max_n = std::max(plan->max_n, n);
    plan->max_tv = std::max(plan->max_tv, tv);
    plan->max_tb = std::max(plan->max_tb, tb);
    plan->h_parts.push_back(pd);
  }
  plan->step_fmas = step_fmas;
  // register-resident fragment plan (sigb_frag.cuh) for the generic path
  {
    FragHost fh;
    std::string why;
    if (plan_fragments(t, fh, why) && frag::supported(fh.NC, fh.G, fh.K)) {
      FragDevPlan& fp = plan->frag;
      fp.NC = fh.NC; fp.G = fh.G; fp.K = fh.K; fp.F = fh.F; fp.cpp = fh.cpp; fp.Fp = fh.Fp;
      fp.pstride = fh.pstride;
      int rc2;
      auto up = [&](auto** dst, const auto& src) -> int {
        using E = typename std::remove_reference<decltype(src)>::type::value_type;
        SIGB_CUDA_TRY(cudaMalloc((void**)dst, sizeof(E) * std::max<size_t>(src.size(), 1)));
        if (!src.empty())
          SIGB_CUDA_TRY(cudaMemcpyAsync((void*)*dst, src.data(), sizeof(E) * src.size(), cudaMemcpyHostToDevice, stream));
        return SIGB_OK;
      };
      if ((rc2 = up(&fp.letter, fh.letter)) || (rc2 = up(&fp.cidx, fh.cidx)) || (rc2 = up(&fp.eidx, fh.eidx)) ||
          (rc2 = up(&fp.sidx, fh.sidx)) || (rc2 = up(&fp.pos, fh.pos)) || (rc2 = up(&fp.red_off, fh.red_off))) {
        sigb_plan_destroy(plan);
        return rc2;
      }
      fp.ok = true;
    }
  }
  // word-set-specialised kernels (sigb_jit.cu): generated lazily, compiled on first use
  if (jit::eligible(t)) {
    plan->jit.eligible = true;
    plan->jit.trie = t;
    jit::make_plan(t, plan->jit.host);
  }
  // perm is stored per part at node_off (same offsets as the node tables)
  auto upload = [&](auto** dst, const auto& src) -> int {
    using E = typename std::remove_reference<decltype(src)>::type::value_type;
    size_t bytes = sizeof(E) * std::max<size_t>(src.size(), 1);
    SIGB_CUDA_TRY(cudaMalloc((void**)dst, bytes));
    if (!src.empty())
      SIGB_CUDA_TRY(cudaMemcpyAsync((void*)*dst, src.data(), sizeof(E) * src.size(), cudaMemcpyHostToDevice, stream));
    return SIGB_OK;
  };
  int rc;
  if ((rc = upload(&plan->d_parts, plan->h_parts)) || (rc = upload(&plan->d_nodeA, nodeA)) ||
      (rc = upload(&plan->d_nodeB, nodeB)) || (rc = upload(&plan->d_perm, perm)) ||
      (rc = upload(&plan->d_lseg, lseg))) {
    sigb_plan_destroy(plan);
    return rc;
  }
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) { sigb_plan_destroy(plan); return cuda_fail(e, "plan upload"); }
  *plan_out = plan;
  return SIGB_OK;
}

extern "C" int sigb_plan_destroy(sigb_plan* plan) {
  if (!plan) return SIGB_OK;
  DeviceGuard guard(plan->device);
  cudaFree(plan->d_parts);
  cudaFree(plan->d_nodeA);
  cudaFree(plan->d_nodeB);
  cudaFree(plan->d_perm);
  cudaFree(plan->d_lseg);
  cudaFree(plan->frag.letter);
  cudaFree(plan->frag.cidx);
  cudaFree(plan->frag.eidx);
  cudaFree(plan->frag.sidx);
  cudaFree(plan->frag.pos);
  cudaFree(plan->frag.red_off);
  for (auto& row : plan->jit.lib)
    for (void* lib : row)
      if (lib) cudaLibraryUnload((cudaLibrary_t)lib);
  delete plan;
  return SIGB_OK;
}

extern "C" int64_t sigb_plan_closure_size(const sigb_plan* plan) { return plan ? plan->Wc : -1; }
extern "C" int64_t sigb_plan_num_parts(const sigb_plan* plan) { return plan ? plan->num_parts : -1; }
extern "C" int64_t sigb_plan_step_fmas(const sigb_plan* plan) { return plan ? plan->step_fmas : -1; }

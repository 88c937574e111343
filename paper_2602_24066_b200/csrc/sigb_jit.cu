// Word-set-specialised Chen kernels for SMALL tries (e.g. config 3's user set):
// a code generator emits straight-line CUDA for every subtree of the closure,
// NVRTC compiles it for sm_100a once per (word set, dtype), and the kernels run
// with LANE = PATH, WARP = TASK:
//   - a task is a few sibling subtrees plus the chain of their common parent's
//     ancestors; every node value, Horner partial and adjoint of the task is a
//     named register in the generated code -- no shared-memory state, no
//     barriers inside a step, no dead slots, and the scaled increments
//     dX[z] / r are computed once per (letter, r) the task uses;
//   - the 32 lanes of a warp run the same task for 32 paths, so the code is
//     warp-uniform; increments are staged per chunk as [step][letter][lane].
// The fragment kernels (sigb_frag.cuh) pay ~24 issue slots of replicated
// chain and dead letter slots per ~7 words on such sets; here every closure
// node is one FMA per target per step.
//
// Backward: per step the task rebuilds its internal nodes
// with -dX, recomputes their partials, runs reverse mode in reverse
// topological order and accumulates dL/d(dX_j) per letter in lane registers;
// the 8 warps (tasks) of a CTA are summed in shared memory in a fixed order
// every kRed steps and the CTA groups of a path by the sample-grads epilogue.
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <sys/stat.h>

#include "sigb_internal.h"

namespace sigb {
namespace jit {

constexpr int kWarps = 4;     // tasks (warps) per CTA
// steps staged per chunk / per CTA gradient reduction (fp64 halves both: smem)
int chunk_steps(int dtype) { return dtype == SIGB_F32 ? 8 : 8; }
int red_steps(int dtype) { return dtype == SIGB_F32 ? 2 : 2; }
constexpr int kCapFwd = 96;   // T-nodes per task, forward
constexpr int kCapBwd = 40;   // T-nodes per task, backward (adjoints double the live values)

namespace {

int64_t tnodes(const Trie& t, int64_t u) { return t.md[u] - t.len[u] + 1; }

int64_t subtree_cost(const Trie& t, int64_t u, std::vector<int64_t>& memo) {
  if (memo[u] >= 0) return memo[u];
  int64_t c = tnodes(t, u);
  for (int64_t k = t.child_first[u]; k < t.child_first[u] + t.child_count[u]; ++k) c += subtree_cost(t, k, memo);
  return memo[u] = c;
}

void subtree(const Trie& t, int64_t u, std::vector<int64_t>& out) {
  out.push_back(u);
  for (int64_t k = t.child_first[u]; k < t.child_first[u] + t.child_count[u]; ++k) subtree(t, k, out);
}

// Units = subtrees of cost <= cap (a larger subtree is split into its
// children's units and its root becomes chain); units of the same parent are
// packed into tasks up to cap.
std::vector<Task> make_tasks(const Trie& t, int64_t cap) {
  const int64_t Wc = (int64_t)t.code.size();
  std::vector<int64_t> memo(Wc, -1);
  std::vector<Task> tasks;
  std::function<void(int64_t, const std::vector<int64_t>&, int64_t, int64_t)> visit =
      [&](int64_t parent, const std::vector<int64_t>& chain, int64_t cf, int64_t cc) {
        std::vector<int64_t> small;
        for (int64_t c = cf; c < cf + cc; ++c) {
          if (subtree_cost(t, c, memo) > cap && t.child_count[c] > 0) {
            std::vector<int64_t> ch2 = chain;
            ch2.push_back(c);
            visit(c, ch2, t.child_first[c], t.child_count[c]);
          } else {
            small.push_back(c);
          }
        }
        (void)parent;
        // chain cost: each chain node evaluates targets up to the deepest level below
        int64_t acc = 0;
        Task cur;
        auto flush = [&]() {
          if (cur.nodes.empty()) return;
          Task tk;
          tk.nodes = chain;
          tk.chain = (int)chain.size();
          tk.nodes.insert(tk.nodes.end(), cur.nodes.begin(), cur.nodes.end());
          tasks.push_back(std::move(tk));
          cur.nodes.clear();
          acc = 0;
        };
        for (int64_t c : small) {
          const int64_t sc = subtree_cost(t, c, memo);
          if (acc > 0 && acc + sc > cap) flush();
          subtree(t, c, cur.nodes);
          acc += sc;
        }
        flush();
      };
  int64_t n1 = 0;
  while (n1 < Wc && t.len[n1] == 1) ++n1;
  visit(-1, {}, 0, n1);
  // similar costs side by side: a CTA's warps wait for each other once per chunk
  auto cost = [&](const Task& tk) {
    int64_t c = 0;
    for (int64_t u : tk.nodes) c += tnodes(t, u);
    return c;
  };
  std::stable_sort(tasks.begin(), tasks.end(), [&](const Task& a, const Task& b) { return cost(a) > cost(b); });
  return tasks;
}

const char* tname(int dtype) { return dtype == SIGB_F32 ? "float" : "double"; }

std::string lit(double v, int dtype) {
  char b[64];
  snprintf(b, sizeof b, dtype == SIGB_F32 ? "%.9gf" : "%.17g", v);
  std::string s = b;
  if (s.find('.') == std::string::npos && s.find('e') == std::string::npos && s.find("inf") == std::string::npos) {
    if (dtype == SIGB_F32) s.insert(s.size() - 1, ".0");
    else s += ".0";
  }
  return s;
}

struct TaskView {
  const Trie& t;
  const Task& tk;
  std::map<int64_t, int> loc;   // closure index -> local id
  std::vector<int> par;         // local parent (-1: empty word)
  std::vector<int> lvl, mdt;    // level, deepest target within the task
  std::vector<std::vector<int>> kids;
  std::set<std::pair<int, int>> scaled;  // (letter, r >= 2) used
  std::set<int> letters;
  TaskView(const Trie& t_, const Task& tk_) : t(t_), tk(tk_) {
    const int n = (int)tk.nodes.size();
    for (int i = 0; i < n; ++i) loc[tk.nodes[i]] = i;
    par.assign(n, -1);
    lvl.assign(n, 0);
    mdt.assign(n, 0);
    kids.assign(n, {});
    for (int i = 0; i < n; ++i) {
      const int64_t u = tk.nodes[i];
      lvl[i] = (int)t.len[u];
      auto it = t.parent[u] >= 0 ? loc.find(t.parent[u]) : loc.end();
      par[i] = it == loc.end() ? -1 : it->second;
      if (par[i] >= 0) kids[par[i]].push_back(i);
    }
    for (int i = n - 1; i >= 0; --i) {
      int m = lvl[i];
      for (int c : kids[i]) m = std::max(m, mdt[c]);
      mdt[i] = m;
    }
    for (int i = 0; i < n; ++i) {
      const int z = letter(i);
      letters.insert(z);
      for (int r = 2; r <= mdt[i] - lvl[i] + 1; ++r) scaled.insert({z, r});
    }
  }
  int letter(int i) const { return (int)(t.code[tk.nodes[i]] % (uint64_t)t.d); }
  // factor dX[letter(i)] / r as an expression
  std::string a(int i, int r) const {
    const int z = letter(i);
    return r == 1 ? "x" + std::to_string(z) : "x" + std::to_string(z) + "_" + std::to_string(r);
  }
  // T(parent(i), m) as an expression; T(eps, m) = 1
  std::string tp(int i, int m, const char* pre) const {
    if (par[i] < 0) return "";
    return std::string(pre) + std::to_string(par[i]) + "_" + std::to_string(m);
  }
};

void emit_letters(std::ostringstream& o, const TaskView& v, int dtype, const char* sign) {
  for (int z : v.letters) o << "        const R x" << z << " = " << sign << "dr[" << z << " * 32];\n";
  for (auto& p : v.scaled)
    o << "        const R x" << p.first << "_" << p.second << " = x" << p.first << " * " << lit(1.0 / p.second, dtype)
      << ";\n";
}

// T(u, m) = a * T(parent, m) + s  (parent eps: a + s)
std::string horner(const TaskView& v, int i, int m, const std::string& s, const char* tpre) {
  const std::string ai = v.a(i, m - v.lvl[i] + 1);
  const std::string tpv = v.tp(i, m, tpre);
  return tpv.empty() ? "(" + ai + " + " + s + ")" : "fma(" + ai + ", " + tpv + ", " + s + ")";
}

std::string common_head(int dtype, int d, bool backward) {
  std::ostringstream o;
  o << "typedef " << tname(dtype) << " R;\n";
  o << "#define D " << d << "\n#define CH " << chunk_steps(dtype) << "\n#define WARPS " << kWarps << "\n";
  o << R"(
// Samples of the CTA's 32 paths are copied with cp.async into Xs; diff() turns
// the landed chunk into Dl[s][z][lane] = increment, after which the next chunk's
// copy is issued into Xs and overlaps the chunk's steps.
#define PITCH ((CH + 1) * D + 1)
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ void cp_async(R* dst, const R* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  if (sizeof(R) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void issue(const R* __restrict__ X, long long B, long long L, long long b0, int j0, int cs,
                                      R* __restrict__ Xb) {
  const int rows = (cs + 1) * D;
  for (int i = threadIdx.x; i < 32 * rows; i += blockDim.x) {
    const int p = i / rows, r = i % rows;
    const long long b = b0 + p;
    if (b < B) cp_async(Xb + p * PITCH + r, X + (b * L + j0) * D + r);
    else Xb[p * PITCH + r] = R(0);
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void diff(const R* __restrict__ Xb, int cs, R* __restrict__ Dl) {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int i = threadIdx.x; i < cs * D * 32; i += blockDim.x) {
    const int s = i / (D * 32), z = (i / 32) % D, p = i % 32;
    const R* xs = Xb + p * PITCH;
    Dl[i] = xs[(s + 1) * D + z] - xs[s * D + z];
  }
  __syncthreads();
}
)";
  (void)backward;
  return o.str();
}

std::string gen_forward(const Trie& t, const std::vector<Task>& tasks, int dtype) {
  const int d = (int)t.d;
  std::ostringstream o;
  o << R"(
extern "C" __global__ void __launch_bounds__(32 * WARPS) sigjit_fwd(const R* __restrict__ X, long long B, long long L,
    R* __restrict__ out, long long out_ld, long long out_col0, int include_empty, R* __restrict__ state,
    long long Wc, int nblocks, int groups, int* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* Xs = reinterpret_cast<R*>(smem_raw);  // samples of the next chunk land here while Dl computes
  R* Dl = Xs + 32 * PITCH;
  const int lane = threadIdx.x & 31;
  const long long M = L - 1;
  // persistent CTAs pinned to a task group by SM: an SM's resident warps run the
  // same few task bodies (instruction-cache locality); path blocks of a group are
  // claimed through an atomic counter, then the CTA helps the other groups
  __shared__ int work;
  const int g0 = smid() % groups;
  for (int pass = 0; pass < groups; ++pass) {
   const int g = (g0 + pass) % groups;
   for (;;) {
    if (threadIdx.x == 0) work = atomicAdd(counters + g, 1);
    __syncthreads();
    const int pb = work;
    __syncthreads();
    if (pb >= nblocks) break;
    const int task = g * WARPS + (threadIdx.x >> 5);
    const long long b0 = (long long)pb * 32, b = b0 + lane;
    R* orow = out ? out + b * out_ld + out_col0 : nullptr;
    R* srow = state ? state + b * Wc : nullptr;
    const bool live = b < B;
    if (orow && live && include_empty && task == 0) orow[-1] = R(1);
    switch (task) {
)";
  std::vector<char> owned(t.code.size(), 0);
  std::ostringstream fns;  // one __noinline__ function per task: registers are allocated per task
  for (size_t ti = 0; ti < tasks.size(); ++ti) {
    TaskView v(t, tasks[ti]);
    const int n = (int)tasks[ti].nodes.size();
    o << "  case " << ti << ": ftask_" << ti << "(X, B, L, M, b0, lane, live, orow, srow, Xs, Dl); break;\n";
    std::ostringstream& o2 = fns;
    o2 << "__device__ __noinline__ void ftask_" << ti << "(const R* __restrict__ X, long long B, long long L, "
          "long long M, long long b0, int lane, bool live, R* __restrict__ orow, R* __restrict__ srow, "
          "R* __restrict__ Xs, R* __restrict__ Dl) {\n";
    {
    std::ostringstream& o = o2;
    for (int i = 0; i < n; ++i) o << "    R s" << i << " = R(0);\n";
    o << "    if (M > 0) issue(X, B, L, b0, 0, (int)(M < CH ? M : CH), Xs);\n";
    o << "    for (long long j0 = 0, c = 0; j0 < M; j0 += CH, ++c) {\n";
    o << "      const int cs = (int)(M - j0 < CH ? M - j0 : CH);\n";
    o << "      diff(Xs, cs, Dl);\n";
    o << "      if (j0 + CH < M) issue(X, B, L, b0, (int)(j0 + CH), (int)(M - j0 - CH < CH ? M - j0 - CH : CH), Xs);\n";
    o << "      #pragma unroll 1\n      for (int s = 0; s < cs; ++s) {\n";
    o << "        const R* dr = Dl + s * D * 32 + lane;\n";
    emit_letters(o, v, dtype, "");
    for (int i = 0; i < n; ++i) {
      for (int m = v.lvl[i] + 1; m <= v.mdt[i]; ++m)
        o << "        const R t" << i << "_" << m << " = " << horner(v, i, m, "s" + std::to_string(i), "t") << ";\n";
      o << "        s" << i << " = " << horner(v, i, v.lvl[i], "s" + std::to_string(i), "t") << ";\n";
    }
    o << "      }\n    }\n";
    o << "    if (live) {\n";
    for (int i = 0; i < n; ++i) {
      const int64_t u = tasks[ti].nodes[i];
      if (owned[u]) continue;
      owned[u] = 1;
      if (t.emit[u] >= 0) o << "      if (orow) orow[" << t.emit[u] << "] = s" << i << ";\n";
      o << "      if (srow) srow[" << u << "] = s" << i << ";\n";
    }
    o << "    }\n}\n";
    }
  }
  o << "  default: {\n    if (M > 0) issue(X, B, L, b0, 0, (int)(M < CH ? M : CH), Xs);\n"
       "    for (long long j0 = 0, c = 0; j0 < M; j0 += CH, ++c) {\n"
       "      diff(Xs, (int)(M - j0 < CH ? M - j0 : CH), Dl);\n"
       "      if (j0 + CH < M) issue(X, B, L, b0, (int)(j0 + CH), (int)(M - j0 - CH < CH ? M - j0 - CH : CH), Xs);\n"
       "    }\n  }\n    }\n   }\n  }\n}\n";
  return common_head(dtype, d, false) + fns.str() + o.str();
}

std::string gen_backward(const Trie& t, const std::vector<Task>& tasks, int dtype) {
  const int d = (int)t.d;
  std::ostringstream head, o;
  head << common_head(dtype, d, true);
  head << "#define KRED " << red_steps(dtype) << "\n";
  head << R"(
// Sum the 8 warps' parked gradients of the last `nr` steps (buffer slot r holds
// step jlast - r) into partial[path][group][j][z], fixed order.
__device__ __forceinline__ void flush(const R* __restrict__ G, int nr, long long jlast, long long B, long long b0,
                                      long long M, R* __restrict__ partial, int groups, int g) {
  __syncthreads();
  for (int i = threadIdx.x; i < nr * D * 32; i += blockDim.x) {
    const int r = i / (D * 32), z = (i / 32) % D, p = i % 32;
    R acc = R(0);
    #pragma unroll
    for (int w = 0; w < WARPS; ++w) acc += G[((w * KRED + r) * D + z) * 32 + p];
    const long long b = b0 + p;
    if (b < B) partial[((b * groups + g) * M + (jlast - r)) * D + z] = acc;
  }
  __syncthreads();
}
)";
  o << R"(
extern "C" __global__ void __launch_bounds__(32 * WARPS) sigjit_bwd(const R* __restrict__ X, long long B, long long L,
    const R* __restrict__ Sin, long long s_ld, long long s_col0, const R* __restrict__ gup, long long g_ld,
    long long g_col0, R* __restrict__ partial, int nblocks, int groups, int* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* Xs = reinterpret_cast<R*>(smem_raw);  // samples of the next chunk land here while Dl computes
  R* Dl = Xs + 32 * PITCH;
  R* Gb = Dl + CH * D * 32;  // [warp][KRED][D][32], letters a task never touches stay 0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long M = L - 1;
  R* gmine = Gb + warp * KRED * D * 32 + lane;
  const int nchunks = (int)((M + CH - 1) / CH);
  __shared__ int work;
  const int g0 = smid() % groups;  // see sigjit_fwd: SM-pinned groups, then help the others
  for (int pass = 0; pass < groups; ++pass) {
   const int g = (g0 + pass) % groups;
   __syncthreads();
   for (int i = threadIdx.x; i < WARPS * KRED * D * 32; i += blockDim.x) Gb[i] = R(0);  // new tasks, new letters
   for (;;) {
    if (threadIdx.x == 0) work = atomicAdd(counters + g, 1);
    __syncthreads();
    const int pb = work;
    __syncthreads();
    if (pb >= nblocks) break;
    const int task = g * WARPS + warp;
    const long long b0 = (long long)pb * 32, b = b0 + lane;
    const bool live = b < B;
    const R* srow = Sin + (live ? b : 0) * s_ld + s_col0;
    const R* grow = gup + (live ? b : 0) * g_ld + g_col0;
    switch (task) {
)";
  std::vector<char> owned(t.code.size(), 0);
  std::ostringstream fns;  // one __noinline__ function per task
  for (size_t ti = 0; ti < tasks.size(); ++ti) {
    TaskView v(t, tasks[ti]);
    const int n = (int)tasks[ti].nodes.size();
    o << "  case " << ti << ": btask_" << ti
      << "(X, B, L, M, b0, lane, live, srow, grow, Xs, Dl, Gb, gmine, partial, groups, g, nchunks); break;\n";
    fns << "__device__ __noinline__ void btask_" << ti << "(const R* __restrict__ X, long long B, long long L, "
           "long long M, long long b0, int lane, bool live, const R* __restrict__ srow, const R* __restrict__ grow, "
           "R* __restrict__ Xs, R* __restrict__ Dl, R* __restrict__ Gb, R* __restrict__ gmine, "
           "R* __restrict__ partial, int groups, int g, int nchunks) {\n";
    {
    std::ostringstream& o = fns;
    std::vector<char> own(n, 0);
    for (int i = 0; i < n; ++i) {
      const int64_t u = tasks[ti].nodes[i];
      if (!owned[u]) { owned[u] = 1; own[i] = 1; }
      const bool internal = !v.kids[i].empty();
      if (internal) o << "    R s" << i << " = live ? srow[" << u << "] : R(0);\n";
      if (own[i] && t.emit[u] >= 0) o << "    R l" << i << " = live ? grow[" << t.emit[u] << "] : R(0);\n";
      else o << "    R l" << i << " = R(0);\n";
    }
    o << "    if (nchunks > 0) issue(X, B, L, b0, (nchunks - 1) * CH, (int)(M - (nchunks - 1) * CH), Xs);\n";
    o << "    for (int c = nchunks - 1; c >= 0; --c) {\n";
    o << "      const int j0 = c * CH;\n      const int cs = (int)(M - j0 < CH ? M - j0 : CH);\n";
    o << "      diff(Xs, cs, Dl);\n";
    o << "      if (c > 0) issue(X, B, L, b0, j0 - CH, CH, Xs);\n      int nb = 0;\n";
    o << "      #pragma unroll 1\n      for (int s = cs - 1; s >= 0; --s) {\n";
    o << "        const R* dr = Dl + s * D * 32 + lane;\n";
    emit_letters(o, v, dtype, "");
    // (a) rebuild internal nodes with -dX: tm partials from the parent's tm
    for (int i = 0; i < n; ++i) {
      if (v.kids[i].empty()) continue;
      const std::string si = "s" + std::to_string(i);
      for (int m = v.lvl[i] + 1; m <= v.mdt[i]; ++m) {
        const std::string ai = v.a(i, m - v.lvl[i] + 1), tpv = v.tp(i, m, "q");
        o << "        const R q" << i << "_" << m << " = "
          << (tpv.empty() ? "(" + si + " - " + ai + ")" : "fma(-" + ai + ", " + tpv + ", " + si + ")") << ";\n";
      }
      const std::string ai = v.a(i, 1), tpv = v.tp(i, v.lvl[i], "q");
      o << "        " << si << " = " << (tpv.empty() ? "(" + si + " - " + ai + ")" : "fma(-" + ai + ", " + tpv + ", " + si + ")")
        << ";\n";
    }
    // (b) forward partials from S_{0,t_j}
    for (int i = 0; i < n; ++i) {
      if (v.kids[i].empty()) continue;
      for (int m = v.lvl[i] + 1; m <= v.mdt[i]; ++m)
        o << "        const R t" << i << "_" << m << " = " << horner(v, i, m, "s" + std::to_string(i), "t") << ";\n";
    }
    // (c) reverse, children before parents
    std::map<int, std::string> gsum;  // letter -> expression list
    for (int i = n - 1; i >= 0; --i) {
      const int l = v.lvl[i];
      const std::string li = "l" + std::to_string(i);
      // Tbar(i, m), m > l, from the children: sum a(c, m - l) * Tbar(c, m)
      for (int m = l + 1; m <= v.mdt[i]; ++m) {
        std::string e;
        for (int c : v.kids[i]) {
          if (v.mdt[c] < m) continue;
          const std::string tbc = m == v.lvl[c] ? "l" + std::to_string(c) : "b" + std::to_string(c) + "_" + std::to_string(m);
          const std::string ac = v.a(c, m - v.lvl[c] + 1);
          e = e.empty() ? ac + " * " + tbc : "fma(" + ac + ", " + tbc + ", " + e + ")";
        }
        o << "        const R b" << i << "_" << m << " = " << (e.empty() ? "R(0)" : e) << ";\n";
      }
      // gradient term for letter(i): sum_m Tbar(i, m) T(parent, m) / (m - l + 1)
      std::string g;
      for (int m = l; m <= v.mdt[i]; ++m) {
        const std::string tb = m == l ? li : "b" + std::to_string(i) + "_" + std::to_string(m);
        const std::string tpv = v.tp(i, m, "t");
        const std::string w = m == l ? tb : tb + " * " + lit(1.0 / (m - l + 1), dtype);
        g = g.empty() ? (tpv.empty() ? w : w + " * " + tpv)
                      : (tpv.empty() ? "(" + g + " + " + w + ")" : "fma(" + w + ", " + tpv + ", " + g + ")");
      }
      const int z = v.letter(i);
      o << "        const R g" << i << " = " << g << ";\n";
      gsum[z] = gsum[z].empty() ? "g" + std::to_string(i) : gsum[z] + " + g" + std::to_string(i);
    }
    // adjoints of the node values for the previous step, after every node used
    // this step's lambda_{j+1} as its Tbar(u, |u|)
    for (int i = 0; i < n; ++i)
      for (int m = v.lvl[i] + 1; m <= v.mdt[i]; ++m) o << "        l" << i << " += b" << i << "_" << m << ";\n";
    // (d) park this step's per-letter gradients (untouched letters stay 0)
    for (auto& kv : gsum) o << "        gmine[(nb * D + " << kv.first << ") * 32] = " << kv.second << ";\n";
    o << "        if (++nb == KRED || s == 0) { flush(Gb, nb, j0 + s + nb - 1, B, b0, M, partial, groups, g); nb = 0; }\n";
    o << "      }\n    }\n}\n";
    }
  }
  o << R"(  default: {
    if (nchunks > 0) issue(X, B, L, b0, (nchunks - 1) * CH, (int)(M - (nchunks - 1) * CH), Xs);
    for (int c = nchunks - 1; c >= 0; --c) {
      const int j0 = c * CH;
      const int cs = (int)(M - j0 < CH ? M - j0 : CH);
      diff(Xs, cs, Dl);
      if (c > 0) issue(X, B, L, b0, j0 - CH, CH, Xs);
      int nb = 0;
      for (int s = cs - 1; s >= 0; --s)
        if (++nb == KRED || s == 0) { flush(Gb, nb, j0 + s + nb - 1, B, b0, M, partial, groups, g); nb = 0; }
    }
  }
    }
   }
  }
}
)";
  return head.str() + fns.str() + o.str();
}

}  // namespace

// Small enough for generated code: few nodes (code size, compile time), shallow,
// and an increment chunk of 32 paths that fits shared memory.
bool eligible(const Trie& t) {
  if (getenv("SIGB_DISABLE_JIT")) return false;
  const int64_t Wc = (int64_t)t.code.size();
  return Wc >= 2 && Wc <= 4096 && t.max_len <= 8 && t.d <= 32;
}

// Task cuts for the forward and the backward of a closure.
void make_plan(const Trie& t, JitHost& h) {
  h.fwd_tasks = make_tasks(t, kCapFwd);
  h.bwd_tasks = make_tasks(t, kCapBwd);
}

std::string source(const Trie& t, const JitHost& h, int dtype, bool backward) {
  return backward ? gen_backward(t, h.bwd_tasks, dtype) : gen_forward(t, h.fwd_tasks, dtype);
}

namespace {

size_t smem_bytes(int dtype, int d, bool backward) {
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  const int ch = chunk_steps(dtype), kr = red_steps(dtype);
  size_t n = 32 * ((size_t)(ch + 1) * d + 1) + (size_t)ch * d * 32;
  if (backward) n += (size_t)kWarps * kr * d * 32;
  return n * es;
}

std::string cache_dir() {
  if (const char* e = getenv("SIGB_JIT_CACHE")) return e;
  const char* home = getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/sigkit_b200/jit";
}

void mkdirs(const std::string& path) {
  std::string cur;
  for (size_t i = 0; i < path.size(); ++i) {
    cur += path[i];
    if (path[i] == '/' || i + 1 == path.size()) mkdir(cur.c_str(), 0755);
  }
}

// NVRTC -> cubin for sm_100a (cached on disk by a hash of the source).
int compile(const std::string& src, std::string& cubin) {
  const std::string key = std::to_string(std::hash<std::string>{}(src)) + "_" + std::to_string(src.size());
  const std::string dir = cache_dir(), path = dir + "/" + key + ".cubin";
  {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      cubin.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
      if (!cubin.empty()) return SIGB_OK;
    }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "sigb_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(SIGB_ERR_CUDA, "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "--use_fast_math=false"};
  nvrtcResult rc = nvrtcCompileProgram(prog, 3, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return fail(SIGB_ERR_CUDA, "NVRTC failed: " + log.substr(0, 2000));
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.assign(n, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  mkdirs(dir);
  std::ofstream out(path + ".tmp", std::ios::binary);
  if (out) {
    out.write(cubin.data(), (std::streamsize)cubin.size());
    out.close();
    std::rename((path + ".tmp").c_str(), path.c_str());
  }
  return SIGB_OK;
}

}  // namespace

int ensure(sigb_plan* p, int dtype, bool backward) {
  JitPlan& J = p->jit;
  const int di = dtype == SIGB_F32 ? 0 : 1, bi = backward ? 1 : 0;
  if (J.kern[di][bi]) return SIGB_OK;
  if (J.failed[di][bi]) return fail(SIGB_ERR_UNSUPPORTED, "word-set kernel compilation failed earlier");
  std::string cubin;
  int rc = compile(source(J.trie, J.host, dtype, backward), cubin);
  if (rc != SIGB_OK) {
    J.failed[di][bi] = J.broken = true;
    return rc;
  }
  cudaLibrary_t lib;
  cudaKernel_t kern;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&kern, lib, backward ? "sigjit_bwd" : "sigjit_fwd");
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_bytes(dtype, (int)p->d, backward));
  if (e != cudaSuccess) {
    J.failed[di][bi] = J.broken = true;
    return cuda_fail(e, "loading the word-set kernel");
  }
  J.lib[di][bi] = (void*)lib;
  J.kern[di][bi] = (void*)kern;
  return SIGB_OK;
}

// Persistent grid: every SM filled once (the kernel claims path blocks itself).
unsigned persistent_grid(const void* kern, size_t smem, int64_t work_items) {
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kWarps, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = 2;
  }
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, work_items));
}

int* counters(const sigb_plan* p, int n, cudaStream_t stream) {
  JitPlan& J = const_cast<sigb_plan*>(p)->jit;
  if (J.ncounters < n) {
    if (J.counters) cudaFree(J.counters);
    J.counters = nullptr;
    if (cudaMalloc((void**)&J.counters, sizeof(int) * n) != cudaSuccess) return nullptr;
    J.ncounters = n;
  }
  if (cudaMemsetAsync(J.counters, 0, sizeof(int) * n, stream) != cudaSuccess) return nullptr;
  return J.counters;
}

int forward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, void* out, int64_t out_ld,
            int64_t out_col0, int include_empty, void* state, cudaStream_t stream) {
  if (B == 0) return SIGB_OK;
  int rc = ensure(const_cast<sigb_plan*>(p), dtype, false);
  if (rc) return rc;
  const int di = dtype == SIGB_F32 ? 0 : 1;
  int groups = (int)((p->jit.host.fwd_tasks.size() + kWarps - 1) / kWarps);
  int nblocks = (int)((B + 31) / 32);
  int* ctr = counters(p, groups, stream);
  if (!ctr) return fail(SIGB_ERR_CUDA, "work counters for the word-set kernel");
  long long Bl = B, Ll = L, ld = out_ld, c0 = out_col0, Wc = p->Wc;
  int inc = include_empty;
  void* args[] = {(void*)&X, &Bl, &Ll, &out, &ld, &c0, &inc, &state, &Wc, &nblocks, &groups, &ctr};
  const size_t smem = smem_bytes(dtype, (int)p->d, false);
  const void* kern = (const void*)p->jit.kern[di][0];
  count_launch();
  timing_begin(0, stream);
  SIGB_CUDA_TRY(cudaLaunchKernel(kern, dim3(persistent_grid(kern, smem, (int64_t)groups * nblocks)), dim3(32 * kWarps),
                                 args, smem, stream));
  timing_end(0, stream);
  return SIGB_OK;
}

namespace {
constexpr size_t kPartialBudget = size_t(4) << 30;

int groups_bwd(const sigb_plan* p) { return (int)((p->jit.host.bwd_tasks.size() + kWarps - 1) / kWarps); }

int64_t bwd_chunk(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  const size_t per_path = (dtype == SIGB_F32 ? 4 : 8) * (size_t)groups_bwd(p) * (size_t)(L - 1) * p->d;
  int64_t c = per_path ? (int64_t)(kPartialBudget / per_path) : B;
  c = std::max<int64_t>(32, c - c % 32);
  return std::min<int64_t>(c, B);
}

template <typename T>
__global__ void jit_sample_grads(const T* __restrict__ partial, int64_t Bc, int64_t P, int64_t M, int64_t d,
                                 int64_t b0, T* __restrict__ dX, T* __restrict__ dinc) {
  const int64_t L = M + 1;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Bc * L * d) return;
  const int64_t z = i % d, t = (i / d) % L, bl = i / (d * L);
  auto inc = [&](int64_t j) {
    T s = T(0);
    for (int64_t q = 0; q < P; ++q) s += partial[((bl * P + q) * M + j) * d + z];
    return s;
  };
  T v = T(0);
  if (t >= 1) v += inc(t - 1);
  if (t < M) {
    const T it = inc(t);
    v -= it;
    if (dinc) dinc[((b0 + bl) * M + t) * d + z] = it;
  }
  dX[((b0 + bl) * L + t) * d + z] = v;
}
}  // namespace

size_t backward_workspace(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  return (dtype == SIGB_F32 ? 4 : 8) * (size_t)bwd_chunk(p, dtype, B, L) * groups_bwd(p) * (size_t)(L - 1) * p->d;
}

int backward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream) {
  int rc = ensure(const_cast<sigb_plan*>(p), dtype, true);
  if (rc) return rc;
  const int di = dtype == SIGB_F32 ? 0 : 1;
  const int groups = groups_bwd(p);
  const int64_t M = L - 1, d = p->d;
  const int64_t chunk = bwd_chunk(p, dtype, B, L);
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  if (!work || work_bytes < es * (size_t)chunk * groups * M * d) return fail(SIGB_ERR_DOMAIN, "backward workspace too small");
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t Bc = std::min(chunk, B - b0);
    const char* Xc = (const char*)X + es * (size_t)b0 * L * d;
    const char* Sc = (const char*)S + es * (size_t)b0 * s_ld;
    const char* gc = (const char*)g + es * (size_t)b0 * g_ld;
    long long Bl = Bc, Ll = L, sl = s_ld, s0 = s_col0, gl = g_ld, g0 = g_col0;
    void* Xv = (void*)Xc;
    void* Sv = (void*)Sc;
    void* gv = (void*)gc;
    int grp = groups, nblocks = (int)((Bc + 31) / 32);
    int* ctr = counters(p, groups, stream);
    if (!ctr) return fail(SIGB_ERR_CUDA, "work counters for the word-set kernel");
    void* args[] = {&Xv, &Bl, &Ll, &Sv, &sl, &s0, &gv, &gl, &g0, &work, &nblocks, &grp, &ctr};
    const size_t smem = smem_bytes(dtype, (int)d, true);
    const void* kern = (const void*)p->jit.kern[di][1];
    count_launch(2);
    timing_begin(1, stream);
    SIGB_CUDA_TRY(cudaLaunchKernel(kern, dim3(persistent_grid(kern, smem, (int64_t)groups * nblocks)),
                                   dim3(32 * kWarps), args, smem, stream));
    timing_end(1, stream);
    const int64_t n = Bc * L * d;
    if (dtype == SIGB_F32)
      jit_sample_grads<float><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>((const float*)work, Bc, groups, M, d, b0,
                                                                             (float*)dX, (float*)dinc);
    else
      jit_sample_grads<double><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>((const double*)work, Bc, groups, M, d,
                                                                              b0, (double*)dX, (double*)dinc);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

}  // namespace jit
}  // namespace sigb

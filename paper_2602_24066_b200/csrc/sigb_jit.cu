// Word-set-specialised Chen kernels for SMALL tries (e.g. config 3's user set):
// a code generator emits straight-line CUDA for every subtree of the closure,
// NVRTC compiles it for sm_100a once per (word set, dtype), and the kernels run
// with LANE = PATH, WARP = TASK:
//   - a task is a few sibling subtrees plus the chain of their common parent's
//     ancestors; every node value, Horner partial and adjoint of the task is a
//     named register in the generated code -- no shared-memory state, no
//     barriers inside a step, no dead slots; the 1/r of the Horner steps
//     rides on the parent's partials (one scale per parent partial, shared
//     by its children and the gradient terms), so a T-node is one FFMA;
//   - the warps of a CTA run different tasks on the same 32 paths.  The CTA's
//     samples arrive per chunk of CH steps by bulk copies (cp.async.bulk, one
//     row of (CH+1)*D samples per path, completion on an mbarrier) and are
//     differenced once into Dl[step][letter][lane] with vector loads, so every
//     task reads an increment with one conflict-free LDS.
// The fragment kernels (sigb_frag.cuh) pay ~24 issue slots of replicated
// chain and dead letter slots per ~7 words on such sets; here every closure
// node is one FMA per target per step.
//
// Backward: per step the task rebuilds its internal nodes
// with -dX, recomputes their partials, runs reverse mode in reverse
// topological order and accumulates dL/d(dX_j) per letter in lane registers
// (one FFMA per T-node against the parent's scaled partial); each warp parks its per-letter
// gradients of the chunk in shared memory and the CTA sums its warps in a
// fixed order once per chunk, behind the barrier the chunk staging needs
// anyway.  Partials [group][step][letter][path] are summed over groups and
// telescoped into dL/dX by jit_sample_grads.
#include <dlfcn.h>
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

#include <atomic>
#include <thread>

#include "sigb_internal.h"

namespace sigb {
namespace jit {

size_t smem_bytes(int dtype, int d, const Cfg& c, bool backward);

namespace {

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// Defaults measured on B200 for config 3 (r01 sweeps, tools/jit_sweep.py):
// the forward runs 3 slots x 4 tasks per SM (12 warps, 168 registers, 16-step
// chunks, 112-T-node tasks: 0.85 -> 0.75 ms against 12 / 96), the
// backward 2 slots x 4 tasks (8 warps, up to 255 registers for 96-T-node
// tasks).  Two slots of the same task on one SM scheduler share its
// instruction cache; separate CTAs of different groups thrash it.
// SIGB_JIT_* override the shape for sweeps; the chunk and slot counts then
// shrink until the CTA fits in shared memory.
Cfg default_cfg(int dtype, int d, bool backward) {
  Cfg c;
  if (!backward) {
    c.warps = env_int("SIGB_JIT_FWARPS", 4);
    c.ch = env_int("SIGB_JIT_FCH", 16);
    c.minb = env_int("SIGB_JIT_FMINB", 1);
    c.cap = env_int("SIGB_JIT_FCAP", 112);
    c.pb = env_int("SIGB_JIT_FPB", 3);
    c.lock = env_int("SIGB_JIT_FLOCK", 0);
    c.maxreg = env_int("SIGB_JIT_FMAXREG", 0);
  } else {
    c.warps = env_int("SIGB_JIT_BWARPS", 4);
    c.ch = env_int("SIGB_JIT_BCH", 8);
    c.minb = env_int("SIGB_JIT_BMINB", 1);
    c.cap = env_int("SIGB_JIT_BCAP", 96);
    c.pb = env_int("SIGB_JIT_BPB", 2);
    c.lock = env_int("SIGB_JIT_BLOCK", 1);
    c.maxreg = env_int("SIGB_JIT_BMAXREG", 184);  // measured best on config 3 (2.98 vs 3.12 ms uncapped)
  }
  c.warps = std::min(std::max(c.warps, 1), 16);
  c.ch = std::min(std::max(c.ch, 1), 64);
  c.minb = std::min(std::max(c.minb, 1), 16);
  c.cap = std::max<int64_t>(c.cap, 1);
  c.pb = std::min(std::max(c.pb, 1), 8);
  c.warps = std::min(c.warps, 32 / c.pb);
  constexpr size_t kSmemMax = 227 * 1024 - 1024;
  while (smem_bytes(dtype, d, c, backward) > kSmemMax && (c.pb > 1 || c.ch > 1)) {
    if (c.ch > 4 || c.pb == 1) c.ch = std::max(1, c.ch / 2);
    else --c.pb;
  }
  return c;
}

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
  std::function<void(const std::vector<int64_t>&, int64_t, int64_t)> visit =
      [&](const std::vector<int64_t>& chain, int64_t cf, int64_t cc) {
        std::vector<int64_t> small;
        for (int64_t c = cf; c < cf + cc; ++c) {
          if (subtree_cost(t, c, memo) > cap && t.child_count[c] > 0) {
            std::vector<int64_t> ch2 = chain;
            ch2.push_back(c);
            visit(ch2, t.child_first[c], t.child_count[c]);
          } else {
            small.push_back(c);
          }
        }
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
  visit({}, 0, n1);
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
    for (int i = 0; i < n; ++i) letters.insert(letter(i));
  }
  int letter(int i) const { return (int)(t.code[tk.nodes[i]] % (uint64_t)t.d); }
  std::string x(int i) const { return "x" + std::to_string(letter(i)); }
  // P(parent(i), m) = T(parent(i), m) / (m - |parent(i)|), the factor of
  // dX[letter(i)] in T(i, m) = dX[letter(i)] / (m - |i| + 1) * T(parent(i), m) + S(i):
  // the 1/r of Alg. 1 moves onto the parent, one scale per parent partial
  // shared by all its children (and by the gradient terms).  T(eps, m) = 1.
  std::string pp(int i, int m, const char* pre, int dtype) const {
    const int pi = par[i];
    if (pi < 0) return lit(1.0 / m, dtype);
    const std::string nm = std::string(pre) + std::to_string(pi) + "_" + std::to_string(m);
    return m - lvl[pi] == 1 ? nm : "p" + nm;
  }
};

void emit_letters(std::ostringstream& o, const TaskView& v) {
  for (int z : v.letters) o << "        const R x" << z << " = dr[" << z << " * 32];\n";
}

// Partials T(i, m), m in (|i|, deepest], named <pre>i_m, and their scaled
// copies p<pre>i_m for r = m - |i| >= 2; then S(i) <- T(i, |i|).  neg: the
// group inverse exp(-dX) of the backward's reconstruction.
void emit_node(std::ostringstream& o, const TaskView& v, int i, const char* pre, bool neg, bool update, int dtype) {
  const std::string si = "s" + std::to_string(i), xi = (neg ? "-" : "") + v.x(i);
  const int l = v.lvl[i];
  if (!v.kids[i].empty())
    for (int m = l + 1; m <= v.mdt[i]; ++m) {
      const std::string nm = std::string(pre) + std::to_string(i) + "_" + std::to_string(m);
      o << "        const R " << nm << " = fma(" << xi << ", " << v.pp(i, m, pre, dtype) << ", " << si << ");\n";
      if (m - l >= 2) o << "        const R p" << nm << " = " << nm << " * " << lit(1.0 / (m - l), dtype) << ";\n";
    }
  if (update) o << "        " << si << " = fma(" << xi << ", " << v.pp(i, l, pre, dtype) << ", " << si << ");\n";
}

double inv_fact(int k) {
  double f = 1;
  for (int i = 2; i <= k; ++i) f *= i;
  return 1.0 / f;
}

// Backward form: Q(i, m) = T(i, m) / (m - |i|)!, so that
//   Q(i, m) = dX[z_i] Q(parent, m) + S(i) / (m - |i|)!,   Q(eps, m) = 1 / m!,
// and with the unscaled adjoints U(i, m) = (m - |i|)! Tbar(i, m),
//   U(i, m) = sum_c dX[z_c] U(c, m),  U(i, |i|) = lambda(i),
//   dL/dX[z] = sum over nodes u of letter z, m of U(u, m) Q(parent(u), m):
// no scale on adjoint or gradient terms, one per state copy S(i) / k!, k >= 2.
std::string qp(const TaskView& v, int i, int m, const char* pre, int dtype) {
  const int pi = v.par[i];
  if (pi < 0) return lit(inv_fact(m), dtype);
  return std::string(pre) + std::to_string(pi) + "_" + std::to_string(m);
}
void emit_node_q(std::ostringstream& o, const TaskView& v, int i, const char* pre, bool neg, bool update, int dtype) {
  const std::string si = "s" + std::to_string(i), xi = (neg ? "-" : "") + v.x(i);
  const int l = v.lvl[i];
  if (!v.kids[i].empty())
    for (int m = l + 1; m <= v.mdt[i]; ++m) {
      const std::string nm = std::string(pre) + std::to_string(i) + "_" + std::to_string(m);
      std::string sc = si;
      if (m - l >= 2) {
        sc = "c" + nm;
        o << "        const R " << sc << " = " << si << " * " << lit(inv_fact(m - l), dtype) << ";\n";
      }
      o << "        const R " << nm << " = fma(" << xi << ", " << qp(v, i, m, pre, dtype) << ", " << sc << ");\n";
    }
  if (update) o << "        " << si << " = fma(" << xi << ", " << qp(v, i, l, pre, dtype) << ", " << si << ");\n";
}

// Vector width of the staging loads/stores and the padded row pitch of the
// sample buffer: rows start 16-byte aligned (bulk-copy destinations) and
// PITCH / VW is odd, so a warp's vector loads of 32 rows hit distinct banks.
int vec_width(int dtype, int d) {
  if (dtype == SIGB_F32) return d % 4 == 0 ? 4 : d % 2 == 0 ? 2 : 1;
  return d % 2 == 0 ? 2 : 1;
}
int pitch(int dtype, int d, int ch) {
  const int es = dtype == SIGB_F32 ? 4 : 8;
  const int al = 16 / es;  // elements per 16 bytes
  int p = (ch + 1) * d;
  p = (p + al - 1) / al * al;
  const int vw = vec_width(dtype, d);
  if ((p / vw) % 2 == 0) p += al;
  return p;
}

std::string common_head(int dtype, int d, const Cfg& c) {
  std::ostringstream o;
  const int vw = vec_width(dtype, d);
  o << "typedef " << tname(dtype) << " R;\n";
  o << "#define D " << d << "\n#define CH " << c.ch << "\n#define WARPS " << c.warps << "\n#define NT (32 * WARPS)\n";
  o << "#define PB " << c.pb << "\n#define LOCK " << c.lock << "\n";
  if (c.maxreg > 0) o << "// maxrregcount " << c.maxreg << "\n";
  o << "#define MINB " << c.minb << "\n#define VW " << vw << "\n#define PITCH " << pitch(dtype, d, c.ch) << "\n";
  o << R"(
struct __align__(VW * sizeof(R)) RV { R v[VW]; };
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned phase) {
  unsigned done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(su32(m)), "r"(phase) : "memory");
  } while (!done);
  __syncwarp();  // lanes may leave the spin at different polls: reconverge before the (aligned) barriers
}
__device__ __forceinline__ int stid() { return (int)threadIdx.x % (32 * WARPS); }  // thread index in the slot
__device__ __forceinline__ int slot_id() { return (int)(threadIdx.x >> 5) / WARPS; }
// LOCK: the slots of a CTA claim their path blocks together and share the
// CTA barrier, so the warps of one task on an SM scheduler stay in lockstep
// (one instruction fetch serves both); otherwise each slot has its own
// named barrier and runs free.
// Non-.aligned barriers: the warps of a slot reach them from different task
// functions (different PCs), which bar.sync / __syncthreads (.aligned) forbid.
__device__ __forceinline__ void slot_sync() {
#if LOCK
  asm volatile("barrier.sync 0;" ::: "memory");
#else
  asm volatile("barrier.sync %0, %1;" ::"r"(1 + slot_id()), "r"(32 * WARPS) : "memory");
#endif
}
__device__ __forceinline__ void cp_async(R* dst, const R* src) {
  if (sizeof(R) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(dst)), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst)), "l"(src) : "memory");
}
// Samples j0 .. j0+cs of the block's 32 paths -> Xs[p * PITCH + s * D + z].
// bulk: one cp.async.bulk per path row (16-byte aligned rows), completion
// counted in bytes on the mbarrier; otherwise element cp.async.
__device__ __forceinline__ void issue(const R* __restrict__ X, long long B, long long L, long long b0, long long j0,
                                      int cs, R* __restrict__ Xs, unsigned long long* mbar, int bulk) {
  const int rows = (cs + 1) * D;
  const long long nl = B - b0 < 32 ? (B > b0 ? B - b0 : 0) : 32;
  if (bulk) {
    if (stid() < 32) {
      const int p = stid();
      if (p == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mbar)),
                     "r"((unsigned)(nl * rows * sizeof(R))) : "memory");
      __syncwarp();
      if (p < nl)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(Xs + p * PITCH)), "l"(X + ((b0 + p) * L + j0) * D), "r"((unsigned)(rows * sizeof(R))),
                     "r"(su32(mbar)) : "memory");
    }
  } else {
    for (int p = stid() >> 5; p < nl; p += WARPS) {
      const R* src = X + ((b0 + p) * L + j0) * D;
      for (int r = stid() & 31; r < rows; r += 32) cp_async(Xs + p * PITCH + r, src + r);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
}
// Wait for the chunk issued last (every thread calls this once per chunk).
__device__ __forceinline__ void land(unsigned long long* mbar, unsigned phase, int bulk) {
  if (bulk) mbar_wait(mbar, phase);
  else asm volatile("cp.async.wait_group 0;" ::: "memory");
}
// Dl[s][z][lane] = X[s+1][z] - X[s][z] for the lane's path.
__device__ __forceinline__ void diff(const R* __restrict__ Xs, int cs, R* __restrict__ Dl) {
  const int lane = threadIdx.x & 31;
  const R* xs = Xs + lane * PITCH;
  for (int it = stid() >> 5; it < cs * (D / VW); it += WARPS) {
    const int s = it / (D / VW), q = it - s * (D / VW);
    const RV a = *reinterpret_cast<const RV*>(xs + (s + 1) * D + q * VW);
    const RV c = *reinterpret_cast<const RV*>(xs + s * D + q * VW);
    R* dl = Dl + (s * D + q * VW) * 32 + lane;
    #pragma unroll
    for (int k = 0; k < VW; ++k) dl[k * 32] = a.v[k] - c.v[k];
  }
}
// A CTA is PB independent slots of WARPS warps (one path block each, own
// named barrier, mbarrier and shared-memory region): the slots share an SM and
// its task group -- the same task bodies in the instruction cache -- but never
// wait for each other.
__device__ __forceinline__ void cta_init(R* base, size_t elems, unsigned long long* mbar) {
  if (threadIdx.x < PB) mbar_init(mbar + threadIdx.x);
  for (size_t i = threadIdx.x; i < elems; i += blockDim.x) base[i] = R(0);  // rows of absent paths stay finite
  __syncthreads();
}
)";
  return o.str();
}

std::string gen_forward(const Trie& t, const std::vector<Task>& tasks, int dtype, const Cfg& cfg) {
  const int d = (int)t.d;
  std::ostringstream o, fns;
  fns << R"(
// Steps of the chunk loop shared by every task body (and the idle warps):
// wait for the chunk, (A) all warps are done with the previous Dl, difference,
// (B) Dl ready and Xs free, prefetch the next chunk into Xs.
#define FWD_CHUNK_BEGIN                                                              \
  const int cs = (int)(M - j0 < CH ? M - j0 : CH);                                   \
  land(mbar, phase, bulk);                                                           \
  phase ^= 1u;                                                                       \
  slot_sync();                                                                       \
  diff(Xs, cs, Dl);                                                                  \
  slot_sync();                                                                       \
  if (j0 + CH < M) issue(X, B, L, b0, j0 + CH, (int)(M - j0 - CH < CH ? M - j0 - CH : CH), Xs, mbar, bulk);
__device__ __noinline__ void fidle(const R* __restrict__ X, long long B, long long L, long long M, long long b0,
                                   R* __restrict__ Xs, R* __restrict__ Dl, unsigned long long* mbar, unsigned phase,
                                   int bulk) {
  if (M > 0) issue(X, B, L, b0, 0, (int)(M < CH ? M : CH), Xs, mbar, bulk);
  for (long long j0 = 0; j0 < M; j0 += CH) { FWD_CHUNK_BEGIN }
}
)";
  o << R"(
extern "C" __global__ void __launch_bounds__(NT * PB, MINB) sigjit_fwd(const R* __restrict__ X, long long B, long long L,
    R* __restrict__ out, long long out_ld, long long out_col0, int include_empty, R* __restrict__ state,
    long long Wc, int nblocks, int groups, int* __restrict__ counters, int bulk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr size_t SLOT = 32 * PITCH + CH * D * 32;
  R* Xs = reinterpret_cast<R*>(smem_raw) + slot_id() * SLOT;
  R* Dl = Xs + 32 * PITCH;
  __shared__ unsigned long long mbars[PB];
  __shared__ int works[PB];
  cta_init(reinterpret_cast<R*>(smem_raw), PB * SLOT, mbars);
  unsigned long long* mbar = mbars + slot_id();
  const int lane = threadIdx.x & 31;
  const long long M = L - 1;
  const unsigned nch = (unsigned)((M + CH - 1) / CH);
  unsigned phase = 0;
  // persistent CTAs pinned to a task group by SM: an SM's resident warps run the
  // same few task bodies (instruction-cache locality); path blocks of a group are
  // claimed through an atomic counter, then the slot helps the other groups
  const int g0 = smid() % groups;
  for (int pass = 0; pass < groups; ++pass) {
   const int g = (g0 + pass) % groups;
   for (;;) {
#if LOCK
    if (threadIdx.x == 0) works[0] = atomicAdd(counters + g, PB);
    __syncthreads();
    const int pbase = works[0];
    __syncthreads();
    if (pbase >= nblocks) break;
    const int pb = pbase + slot_id();
    const int task = pb < nblocks ? g * WARPS + (threadIdx.x >> 5) % WARPS : 0x7fffffff;  // idle slot
#else
    if (stid() == 0) works[slot_id()] = atomicAdd(counters + g, 1);
    slot_sync();
    const int pb = works[slot_id()];
    slot_sync();
    if (pb >= nblocks) break;
    const int task = g * WARPS + (threadIdx.x >> 5) % WARPS;
#endif
    const long long b0 = (long long)pb * 32, b = b0 + lane;
    const bool live = b < B;
    R* orow = out && live ? out + b * out_ld + out_col0 : nullptr;
    R* srow = state && live ? state + b * Wc : nullptr;
    if (orow && include_empty && task == 0) orow[-1] = R(1);
    switch (task) {
)";
  std::vector<char> owned(t.code.size(), 0);
  for (size_t ti = 0; ti < tasks.size(); ++ti) {
    TaskView v(t, tasks[ti]);
    const int n = (int)tasks[ti].nodes.size();
    o << "  case " << ti << ": ftask_" << ti << "(X, B, L, M, b0, orow, srow, Xs, Dl, mbar, phase, bulk); break;\n";
    fns << "__device__ __noinline__ void ftask_" << ti << "(const R* __restrict__ X, long long B, long long L, "
           "long long M, long long b0, R* __restrict__ orow, R* __restrict__ srow, R* __restrict__ Xs, "
           "R* __restrict__ Dl, unsigned long long* mbar, unsigned phase, int bulk) {\n";
    fns << "  const int lane = threadIdx.x & 31;\n";
    for (int i = 0; i < n; ++i) fns << "  R s" << i << " = R(0);\n";
    fns << "  if (M > 0) issue(X, B, L, b0, 0, (int)(M < CH ? M : CH), Xs, mbar, bulk);\n";
    fns << "  for (long long j0 = 0; j0 < M; j0 += CH) {\n    FWD_CHUNK_BEGIN\n";
    fns << "    #pragma unroll 1\n    for (int s = 0; s < cs; ++s) {\n";
    fns << "        const R* dr = Dl + s * D * 32 + lane;\n";
    emit_letters(fns, v);
    for (int i = 0; i < n; ++i) emit_node(fns, v, i, "t", false, true, dtype);
    fns << "    }\n  }\n";
    for (int i = 0; i < n; ++i) {
      const int64_t u = tasks[ti].nodes[i];
      if (owned[u]) continue;
      owned[u] = 1;
      if (t.emit[u] >= 0) fns << "  if (orow) orow[" << t.emit[u] << "] = s" << i << ";\n";
      fns << "  if (srow) srow[" << u << "] = s" << i << ";\n";
    }
    fns << "}\n";
  }
  o << "  default: fidle(X, B, L, M, b0, Xs, Dl, mbar, phase, bulk);\n    }\n    phase ^= nch & 1u;\n   }\n  }\n}\n";
  return common_head(dtype, d, cfg) + fns.str() + o.str();
}

std::string gen_backward(const Trie& t, const std::vector<Task>& tasks, int dtype, const Cfg& cfg) {
  const int d = (int)t.d;
  std::ostringstream fns, o;
  fns << R"(
// Sum the warps' parked gradients of one chunk (Gb[warp][s][z][lane], s local)
// into partial[g][j0+s][z][path] (path pitch Bp), fixed warp order.
__device__ __forceinline__ void reduce(const R* __restrict__ Gb, long long j0, int cs, R* __restrict__ partial,
                                       long long Bp, long long M, int g, long long b0) {
  if (b0 >= Bp) return;  // idle slot (LOCK): no paths
  for (int i = stid(); i < cs * D * (32 / VW); i += NT) {
    const int q = i % (32 / VW), sz = i / (32 / VW);
    RV acc = *reinterpret_cast<const RV*>(Gb + sz * 32 + q * VW);
    #pragma unroll
    for (int w = 1; w < WARPS; ++w) {
      const RV t = *reinterpret_cast<const RV*>(Gb + (w * CH * D + sz) * 32 + q * VW);
      #pragma unroll
      for (int k = 0; k < VW; ++k) acc.v[k] += t.v[k];
    }
    const int s = sz / D, z = sz - s * D;
    *reinterpret_cast<RV*>(partial + (((long long)g * M + j0 + s) * D + z) * Bp + b0 + q * VW) = acc;
  }
}
// Chunk prologue of the reverse sweep (every warp, every chunk c = nch-1 .. 0):
// wait for the chunk, (A) every warp is done with chunk c+1 -> sum its parked
// gradients, difference chunk c, (B) Dl ready / Xs and Gb free, prefetch c-1.
#define BWD_CHUNK_BEGIN                                                                     \
  const long long j0 = (long long)c * CH;                                                   \
  const int cs = (int)(M - j0 < CH ? M - j0 : CH);                                          \
  land(mbar, phase, bulk);                                                                  \
  phase ^= 1u;                                                                              \
  slot_sync();                                                                              \
  if (c + 1 < nch) reduce(Gb, j0 + CH, (int)(M - j0 - CH < CH ? M - j0 - CH : CH), partial, Bp, M, g, b0); \
  diff(Xs, cs, Dl);                                                                         \
  slot_sync();                                                                              \
  if (c > 0) issue(X, B, L, b0, j0 - CH, CH, Xs, mbar, bulk);
#define BWD_PROLOGUE                                                                        \
  const int nch = (int)((M + CH - 1) / CH);                                                 \
  if (nch > 0) issue(X, B, L, b0, (long long)(nch - 1) * CH, (int)(M - (long long)(nch - 1) * CH), Xs, mbar, bulk);
#define BWD_EPILOGUE                                                                        \
  slot_sync();                                                                              \
  if (nch > 0) reduce(Gb, 0, (int)(M < CH ? M : CH), partial, Bp, M, g, b0);
__device__ __noinline__ void bidle(const R* __restrict__ X, long long B, long long L, long long M, long long b0,
                                   R* __restrict__ Xs, R* __restrict__ Dl, R* __restrict__ Gb, R* __restrict__ partial,
                                   long long Bp, int g, unsigned long long* mbar, unsigned phase, int bulk) {
  BWD_PROLOGUE
  for (int c = nch - 1; c >= 0; --c) { BWD_CHUNK_BEGIN }
  BWD_EPILOGUE
}
)";
  o << R"(
extern "C" __global__ void __launch_bounds__(NT * PB, MINB) sigjit_bwd(const R* __restrict__ X, long long B, long long L,
    const R* __restrict__ Sin, long long s_ld, long long s_col0, const R* __restrict__ gup, long long g_ld,
    long long g_col0, R* __restrict__ partial, long long Bp, int nblocks, int groups, int* __restrict__ counters,
    int bulk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr size_t SLOT = 32 * PITCH + CH * D * 32 + WARPS * CH * D * 32;
  R* Xs = reinterpret_cast<R*>(smem_raw) + slot_id() * SLOT;
  R* Dl = Xs + 32 * PITCH;
  R* Gb = Dl + CH * D * 32;  // [warp][CH][D][32]; letters a task never touches stay 0
  __shared__ unsigned long long mbars[PB];
  __shared__ int works[PB];
  cta_init(reinterpret_cast<R*>(smem_raw), PB * SLOT, mbars);
  unsigned long long* mbar = mbars + slot_id();
  const int lane = threadIdx.x & 31;
  const long long M = L - 1;
  const unsigned nch = (unsigned)((M + CH - 1) / CH);
  unsigned phase = 0;
  const int g0 = smid() % groups;  // see sigjit_fwd: SM-pinned groups, then help the others
  for (int pass = 0; pass < groups; ++pass) {
   const int g = (g0 + pass) % groups;
   slot_sync();
   for (int i = stid(); i < WARPS * CH * D * 32; i += NT) Gb[i] = R(0);  // new tasks, new letters
   for (;;) {
#if LOCK
    if (threadIdx.x == 0) works[0] = atomicAdd(counters + g, PB);
    __syncthreads();
    const int pbase = works[0];
    __syncthreads();
    if (pbase >= nblocks) break;
    const int pb = pbase + slot_id();
    const int task = pb < nblocks ? g * WARPS + (threadIdx.x >> 5) % WARPS : 0x7fffffff;  // idle slot
#else
    if (stid() == 0) works[slot_id()] = atomicAdd(counters + g, 1);
    slot_sync();
    const int pb = works[slot_id()];
    slot_sync();
    if (pb >= nblocks) break;
    const int task = g * WARPS + (threadIdx.x >> 5) % WARPS;
#endif
    const long long b0 = (long long)pb * 32, b = b0 + lane;
    const bool live = b < B;
    const R* srow = Sin + (live ? b : 0) * s_ld + s_col0;
    const R* grow = gup + (live ? b : 0) * g_ld + g_col0;
    switch (task) {
)";
  std::vector<char> owned(t.code.size(), 0);
  for (size_t ti = 0; ti < tasks.size(); ++ti) {
    TaskView v(t, tasks[ti]);
    const int n = (int)tasks[ti].nodes.size();
    o << "  case " << ti << ": btask_" << ti
      << "(X, B, L, M, b0, live, srow, grow, Xs, Dl, Gb, partial, Bp, g, mbar, phase, bulk); break;\n";
    fns << "__device__ __noinline__ void btask_" << ti << "(const R* __restrict__ X, long long B, long long L, "
           "long long M, long long b0, bool live, const R* __restrict__ srow, const R* __restrict__ grow, "
           "R* __restrict__ Xs, R* __restrict__ Dl, R* __restrict__ Gb, R* __restrict__ partial, long long Bp, "
           "int g, unsigned long long* mbar, unsigned phase, int bulk) {\n";
    fns << "  const int lane = threadIdx.x & 31;\n";
    fns << "  R* gmine = Gb + ((threadIdx.x >> 5) % WARPS) * CH * D * 32 + lane;\n";
    std::vector<char> own(n, 0);
    for (int i = 0; i < n; ++i) {
      const int64_t u = tasks[ti].nodes[i];
      if (!owned[u]) { owned[u] = 1; own[i] = 1; }
      if (!v.kids[i].empty()) fns << "  R s" << i << " = live ? srow[" << u << "] : R(0);\n";
      if (own[i] && t.emit[u] >= 0) fns << "  R l" << i << " = live ? grow[" << t.emit[u] << "] : R(0);\n";
      else fns << "  R l" << i << " = R(0);\n";
    }
    fns << "  BWD_PROLOGUE\n";
    fns << "  for (int c = nch - 1; c >= 0; --c) {\n    BWD_CHUNK_BEGIN\n";
    fns << "    #pragma unroll 1\n    for (int s = cs - 1; s >= 0; --s) {\n";
    fns << "        const R* dr = Dl + s * D * 32 + lane;\n";
    emit_letters(fns, v);
    // (a) rebuild internal nodes with -dX (S_{0,t_j} = S_{0,t_j+1} (x) exp(-dX_j)), top-down
    for (int i = 0; i < n; ++i)
      if (!v.kids[i].empty()) emit_node_q(fns, v, i, "q", true, true, dtype);
    // (b) forward partials from S_{0,t_j}
    for (int i = 0; i < n; ++i)
      if (!v.kids[i].empty()) emit_node_q(fns, v, i, "t", false, false, dtype);
    // (c) reverse, children before parents (U form, see emit_node_q)
    std::set<int> gstarted;
    for (int i = n - 1; i >= 0; --i) {
      const int l = v.lvl[i];
      const std::string li = "l" + std::to_string(i);
      for (int m = l + 1; m <= v.mdt[i]; ++m) {
        std::string e;
        for (int c : v.kids[i]) {
          if (v.mdt[c] < m) continue;
          const std::string tbc = m == v.lvl[c] ? "l" + std::to_string(c) : "b" + std::to_string(c) + "_" + std::to_string(m);
          e = e.empty() ? v.x(c) + " * " + tbc : "fma(" + v.x(c) + ", " + tbc + ", " + e + ")";
        }
        fns << "        const R b" << i << "_" << m << " = " << e << ";\n";
      }
      const int z = v.letter(i);
      const std::string G = "G" + std::to_string(z);
      for (int m = l; m <= v.mdt[i]; ++m) {
        const std::string tb = m == l ? li : "b" + std::to_string(i) + "_" + std::to_string(m);
        const std::string P = qp(v, i, m, "t", dtype);
        if (!gstarted.count(z)) {
          gstarted.insert(z);
          fns << "        R " << G << " = " << tb << " * " << P << ";\n";
        } else {
          fns << "        " << G << " = fma(" << tb << ", " << P << ", " << G << ");\n";
        }
      }
    }
    // adjoints of the node values for the previous step, after every node used
    // this step's lambda_{j+1} as its Tbar(u, |u|)
    for (int i = 0; i < n; ++i)
      for (int m = v.lvl[i] + 1; m <= v.mdt[i]; ++m) {
        if (m - v.lvl[i] == 1) fns << "        l" << i << " += b" << i << "_" << m << ";\n";
        else fns << "        l" << i << " = fma(b" << i << "_" << m << ", " << lit(inv_fact(m - v.lvl[i]), dtype) << ", l" << i << ");\n";
      }
    // (d) park dL/d(dX_j) for the chunk reduction
    for (int z : gstarted) fns << "        gmine[(s * D + " << z << ") * 32] = G" << z << ";\n";
    fns << "    }\n  }\n  BWD_EPILOGUE\n}\n";
  }
  o << "  default: bidle(X, B, L, M, b0, Xs, Dl, Gb, partial, Bp, g, mbar, phase, bulk);\n"
       "    }\n    phase ^= nch & 1u;\n   }\n  }\n}\n";
  return common_head(dtype, d, cfg) + fns.str() + o.str();
}

}  // namespace

// Small enough for generated code: few nodes (code size, compile time), shallow,
// and an increment chunk of 32 paths that fits shared memory.
bool eligible(const Trie& t) {
  if (getenv("SIGB_DISABLE_JIT")) return false;
  const int64_t Wc = (int64_t)t.code.size();
  return Wc >= 2 && Wc <= 4096 && t.max_len <= 8 && t.d <= 32;
}

// Task cuts and launch shapes for the forward and the backward of a closure.
void make_plan(const Trie& t, JitHost& h) {
  for (int di = 0; di < 2; ++di)
    for (int bi = 0; bi < 2; ++bi) h.cfg[di][bi] = default_cfg(di == 0 ? SIGB_F32 : SIGB_F64, (int)t.d, bi == 1);
  h.fwd_tasks = make_tasks(t, h.cfg[0][0].cap);
  h.bwd_tasks = make_tasks(t, h.cfg[0][1].cap);
}

std::string source(const Trie& t, const JitHost& h, int dtype, bool backward) {
  const Cfg& c = h.cfg[dtype == SIGB_F32 ? 0 : 1][backward ? 1 : 0];
  return backward ? gen_backward(t, h.bwd_tasks, dtype, c) : gen_forward(t, h.fwd_tasks, dtype, c);
}

size_t smem_bytes(int dtype, int d, const Cfg& c, bool backward) {
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  size_t n = 32 * (size_t)pitch(dtype, d, c.ch) + (size_t)c.ch * d * 32;
  if (backward) n += (size_t)c.warps * c.ch * d * 32;
  return n * es * c.pb;
}

namespace {

// Cubin cache directories, searched in order: $SIGB_JIT_CACHE alone if set,
// else jit_cache/ next to libsigkit_b200.so (filled by the build for the
// shipped word sets, travels with the tree) and ~/.cache/sigkit_b200/jit.
// New cubins go to the first writable one.
std::vector<std::string> cache_dirs() {
  if (const char* e = getenv("SIGB_JIT_CACHE")) return {e};
  std::vector<std::string> dirs;
  Dl_info info;
  if (dladdr((void*)&cache_dirs, &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const size_t k = so.find_last_of('/');
    dirs.push_back((k == std::string::npos ? std::string(".") : so.substr(0, k)) + "/jit_cache");
  }
  const char* home = getenv("HOME");
  dirs.push_back(std::string(home ? home : "/tmp") + "/.cache/sigkit_b200/jit");
  return dirs;
}

void mkdirs(const std::string& path) {
  std::string cur;
  for (size_t i = 0; i < path.size(); ++i) {
    cur += path[i];
    if (path[i] == '/' || i + 1 == path.size()) mkdir(cur.c_str(), 0755);
  }
}

std::string cache_key(const std::string& src) {
  const char* xo = getenv("SIGB_JIT_NVRTC_OPTS");
  const std::string keysrc = xo ? src + "\n// opts: " + xo : src;
  return std::to_string(std::hash<std::string>{}(keysrc)) + "_" + std::to_string(src.size());
}

// cubin from the on-disk cache, if present
bool cache_lookup(const std::string& src, std::string& cubin) {
  const std::string key = cache_key(src);
  for (const std::string& dir : cache_dirs()) {
    std::ifstream in(dir + "/" + key + ".cubin", std::ios::binary);
    if (in) {
      cubin.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
      if (!cubin.empty()) return true;
    }
  }
  return false;
}

// NVRTC -> cubin for sm_100a (cached on disk by a hash of the source).
int compile(const std::string& src, std::string& cubin) {
  if (cache_lookup(src, cubin)) return SIGB_OK;
  const std::string key = cache_key(src);
  const std::vector<std::string> dirs = cache_dirs();
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "sigb_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(SIGB_ERR_CUDA, "nvrtcCreateProgram failed");
  // SIGB_JIT_NVRTC_OPTS: extra space-separated NVRTC options (sweeps only; part of the cache key)
  std::vector<std::string> extra;
  if (const char* e = getenv("SIGB_JIT_NVRTC_OPTS")) {
    std::istringstream is(e);
    for (std::string w; is >> w;) extra.push_back(w);
  }
  // a register cap chosen by the generator travels in the source ("// maxrregcount N")
  const size_t mr = src.find("// maxrregcount ");
  if (mr != std::string::npos) extra.push_back("--maxrregcount=" + std::to_string(atoi(src.c_str() + mr + 16)));
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "-lineinfo"};
  for (const std::string& w : extra) opts.push_back(w.c_str());
  nvrtcResult rc = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
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
  for (const std::string& dir : dirs) {
    mkdirs(dir);
    const std::string path = dir + "/" + key + ".cubin";
    std::ofstream out(path + ".tmp", std::ios::binary);
    if (!out) continue;
    out.write(cubin.data(), (std::streamsize)cubin.size());
    out.close();
    if (out && std::rename((path + ".tmp").c_str(), path.c_str()) == 0) break;
  }
  return SIGB_OK;
}

const Cfg& cfg_of(const sigb_plan* p, int dtype, bool backward) {
  return p->jit.host.cfg[dtype == SIGB_F32 ? 0 : 1][backward ? 1 : 0];
}

}  // namespace

// Host-only: generate and compile a word set's kernel into the cache (no device).
int precompile(const Trie& t, int dtype, bool backward) {
  JitHost h;
  make_plan(t, h);
  std::string cubin;
  return compile(source(t, h, dtype, backward), cubin);
}

struct Pending {
  std::atomic<int> state{0};  // 0 compiling, 1 cubin ready, 2 failed
  std::string cubin, err;
};

namespace {
// Background compiles still running when the process exits would race NVRTC's own teardown
// (a crash at exit): the library's static destructor -- run before libnvrtc's, which it depends
// on -- waits for them (bounded).
std::atomic<int> g_inflight{0};
struct InflightGuard {
  ~InflightGuard() {
    for (int i = 0; i < 24000 && g_inflight.load(std::memory_order_acquire) > 0; ++i)
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
  }
} g_inflight_guard;
}  // namespace

bool wait_default() {
  static const bool sync_env = getenv("SIGB_JIT_SYNC") && atoi(getenv("SIGB_JIT_SYNC")) != 0;
  return g_policy == 4 || sync_env;
}

namespace {
int load(sigb_plan* p, int dtype, bool backward, const std::string& cubin) {
  JitPlan& J = p->jit;
  const int di = dtype == SIGB_F32 ? 0 : 1, bi = backward ? 1 : 0;
  cudaLibrary_t lib;
  cudaKernel_t kern;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&kern, lib, backward ? "sigjit_bwd" : "sigjit_fwd");
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_bytes(dtype, (int)p->d, cfg_of(p, dtype, backward), backward));
  if (e != cudaSuccess) {
    J.failed[di][bi] = J.broken = true;
    return cuda_fail(e, "loading the word-set kernel");
  }
  J.lib[di][bi] = (void*)lib;
  J.kern[di][bi] = (void*)kern;
  return SIGB_OK;
}
}  // namespace

int ensure(sigb_plan* p, int dtype, bool backward, bool wait) {
  JitPlan& J = p->jit;
  const int di = dtype == SIGB_F32 ? 0 : 1, bi = backward ? 1 : 0;
  std::lock_guard<std::mutex> lock(J.mu);
  if (J.kern[di][bi]) return SIGB_OK;
  if (J.standin[di][bi] && !wait) return kPending;  // a forced wait (policy 4, SIGB_JIT_SYNC) overrides the pin
  if (J.failed[di][bi]) return fail(SIGB_ERR_UNSUPPORTED, "word-set kernel compilation failed earlier");
  std::shared_ptr<Pending>& pd = J.pending[di][bi];
  if (!pd) {
    const std::string src = source(J.trie, J.host, dtype, backward);
    std::string cubin;
    if (cache_lookup(src, cubin)) return load(p, dtype, backward, cubin);
    pd = std::make_shared<Pending>();
    std::shared_ptr<Pending> job = pd;
    // host-only work (no CUDA calls): the thread owns its share of the job and may outlive the plan
    g_inflight.fetch_add(1, std::memory_order_acq_rel);
    std::thread([job, src]() {
      std::string out;
      const int rc = compile(src, out);
      if (rc == SIGB_OK) {
        job->cubin.swap(out);
        job->state.store(1, std::memory_order_release);
      } else {
        job->err = "NVRTC compile of the word-set kernel failed";
        job->state.store(2, std::memory_order_release);
      }
      g_inflight.fetch_sub(1, std::memory_order_acq_rel);
    }).detach();
  }
  if (wait)
    while (pd->state.load(std::memory_order_acquire) == 0) std::this_thread::sleep_for(std::chrono::milliseconds(5));
  const int st = pd->state.load(std::memory_order_acquire);
  if (st == 0) {
    J.standin[di][bi] = true;
    return kPending;
  }
  if (st == 2) {
    J.failed[di][bi] = J.broken = true;
    return fail(SIGB_ERR_UNSUPPORTED, pd->err);
  }
  const int rc = load(p, dtype, backward, pd->cubin);
  pd.reset();
  return rc;
}

namespace {

// Persistent grid: every SM filled once (the kernel claims path blocks itself).
unsigned persistent_grid(const void* kern, int threads, size_t smem, int64_t work_items) {
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = 1;
  }
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, work_items));
}

// Work counters of the persistent kernels are stream-ordered per launch (the
// backward's live in its workspace, the forward's come from cudaMallocAsync), so
// launches of one plan on several streams or threads never share them.
int zero_counters(int* ctr, int n, cudaStream_t stream) {
  SIGB_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(int) * n, stream));
  return SIGB_OK;
}

// Bulk copies need 16-byte aligned rows: D * sizeof(R) and the base pointer.
int bulk_ok(const void* X, int dtype, int64_t d) {
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  return ((uintptr_t)X % 16 == 0 && (d * es) % 16 == 0) ? 1 : 0;
}

}  // namespace

int forward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, void* out, int64_t out_ld,
            int64_t out_col0, int include_empty, void* state, cudaStream_t stream) {
  if (B == 0) return SIGB_OK;
  int rc = ensure(const_cast<sigb_plan*>(p), dtype, false, wait_default());
  if (rc) return rc;
  const int di = dtype == SIGB_F32 ? 0 : 1;
  const Cfg& c = cfg_of(p, dtype, false);
  int groups = (int)((p->jit.host.fwd_tasks.size() + c.warps - 1) / c.warps);
  int nblocks = (int)((B + 31) / 32);
  int* ctr = nullptr;
  SIGB_CUDA_TRY(cudaMallocAsync((void**)&ctr, sizeof(int) * groups, stream));
  if ((rc = zero_counters(ctr, groups, stream))) return rc;
  long long Bl = B, Ll = L, ld = out_ld, c0 = out_col0, Wc = p->Wc;
  int inc = include_empty, bulk = bulk_ok(X, dtype, p->d);
  void* args[] = {(void*)&X, &Bl, &Ll, &out, &ld, &c0, &inc, &state, &Wc, &nblocks, &groups, &ctr, &bulk};
  const size_t smem = smem_bytes(dtype, (int)p->d, c, false);
  const void* kern = (const void*)p->jit.kern[di][0];
  count_launch();
  timing_begin(0, stream);
  const int threads = 32 * c.warps * c.pb;
  const cudaError_t le = cudaLaunchKernel(
      kern, dim3(persistent_grid(kern, threads, smem, ((int64_t)groups * nblocks + c.pb - 1) / c.pb)), dim3(threads),
      args, smem, stream);
  timing_end(0, stream);
  SIGB_CUDA_TRY(cudaFreeAsync(ctr, stream));
  SIGB_CUDA_TRY(le);
  return SIGB_OK;
}

namespace {
constexpr int kTT = 16;  // samples per sample-grads tile

int groups_bwd(const sigb_plan* p, int dtype) {
  const int w = cfg_of(p, dtype, true).warps;
  return (int)((p->jit.host.bwd_tasks.size() + w - 1) / w);
}

int64_t pad32(int64_t n) { return (n + 31) / 32 * 32; }

int64_t bwd_chunk(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  const size_t per_path = (dtype == SIGB_F32 ? 4 : 8) * (size_t)groups_bwd(p, dtype) * (size_t)(L - 1) * p->d;
  int64_t c = per_path ? (int64_t)(partial_budget() / 2 / per_path) : B;
  c = std::min<int64_t>(std::max<int64_t>(32, c - c % 32), int64_t(1) << 20);
  return std::min<int64_t>(c, B);
}

// dX[b][t] = inc(t-1) - inc(t), inc(j)[z] = sum_g partial[g][j][z][b]: a CTA
// sums a tile of 32 paths x (kTT+1) increments (16-byte path-contiguous loads,
// groups unrolled for memory parallelism), then writes the tile's samples row
// by row (each path's kTT*d samples are contiguous in dX).
template <typename T>
__global__ void __launch_bounds__(256) jit_sample_grads(const T* __restrict__ partial, int64_t Bp, int64_t Bc, int P,
                                                        int64_t M, int d, int64_t b0, T* __restrict__ dX,
                                                        T* __restrict__ dinc) {
  constexpr int V = 16 / sizeof(T);  // paths per 16-byte load
  struct __align__(16) Vec { T v[V]; };
  extern __shared__ __align__(16) unsigned char sg_raw[];
  T* inc = reinterpret_cast<T*>(sg_raw);  // [kTT + 1][d][33]
  const int64_t L = M + 1;
  const int64_t pb = (int64_t)blockIdx.y * 32, t0 = (int64_t)blockIdx.x * kTT;
  const int64_t gs = M * d * Bp;
  const int nq = (kTT + 1) * d * (32 / V);
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    const int q = i % (32 / V), r = i / (32 / V);
    const int jj = r / d, z = r - jj * d;
    const int64_t j = t0 - 1 + jj;
    Vec acc;
#pragma unroll
    for (int k = 0; k < V; ++k) acc.v[k] = T(0);
    if (j >= 0 && j < M) {
      const T* src = partial + (j * d + z) * Bp + pb + q * V;
      int g = 0;
      for (; g + 4 <= P; g += 4) {
        const Vec a = *reinterpret_cast<const Vec*>(src + (g + 0) * gs);
        const Vec b = *reinterpret_cast<const Vec*>(src + (g + 1) * gs);
        const Vec c = *reinterpret_cast<const Vec*>(src + (g + 2) * gs);
        const Vec e = *reinterpret_cast<const Vec*>(src + (g + 3) * gs);
#pragma unroll
        for (int k = 0; k < V; ++k) acc.v[k] += a.v[k] + b.v[k] + c.v[k] + e.v[k];
      }
      for (; g < P; ++g) {
        const Vec a = *reinterpret_cast<const Vec*>(src + g * gs);
#pragma unroll
        for (int k = 0; k < V; ++k) acc.v[k] += a.v[k];
      }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) inc[r * 33 + q * V + k] = acc.v[k];
  }
  __syncthreads();
  const int row = kTT * d;
  for (int i = threadIdx.x; i < 32 * row; i += blockDim.x) {
    const int p = i / row, e = i - p * row, tt = e / d, z = e - tt * d;
    const int64_t b = pb + p, t = t0 + tt;
    if (b >= Bc || t >= L) continue;
    const T hi = inc[(tt * d + z) * 33 + p], lo = inc[((tt + 1) * d + z) * 33 + p];
    dX[((b0 + b) * L + t) * d + z] = hi - lo;
    if (dinc && t < M) dinc[((b0 + b) * M + t) * d + z] = lo;
  }
}
}  // namespace

size_t partial_bytes(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  return (dtype == SIGB_F32 ? 4 : 8) * (size_t)pad32(bwd_chunk(p, dtype, B, L)) * groups_bwd(p, dtype) *
         (size_t)(L - 1) * p->d;
}

// partials, then the persistent kernel's work counters (one int per task group)
size_t backward_workspace(const sigb_plan* p, int dtype, int64_t B, int64_t L) {
  return partial_bytes(p, dtype, B, L) + sizeof(int) * (size_t)groups_bwd(p, dtype);
}

int backward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream) {
  int rc = ensure(const_cast<sigb_plan*>(p), dtype, true, wait_default());
  if (rc) return rc;
  const int di = dtype == SIGB_F32 ? 0 : 1;
  const Cfg& c = cfg_of(p, dtype, true);
  const int groups = groups_bwd(p, dtype);
  const int64_t M = L - 1, d = p->d;
  const int64_t chunk = bwd_chunk(p, dtype, B, L);
  const size_t es = dtype == SIGB_F32 ? 4 : 8;
  if (!work || work_bytes < backward_workspace(p, dtype, B, L))
    return fail(SIGB_ERR_DOMAIN, "backward workspace too small");
  int* ctr = (int*)((char*)work + partial_bytes(p, dtype, B, L));
  if ((uintptr_t)work % 16) return fail(SIGB_ERR_DOMAIN, "backward workspace must be 16-byte aligned");
  static bool attr[64][2] = {};  // per device: sample-grads tiles above 48 KB (fp64, large d)
  int devno = 0;
  cudaGetDevice(&devno);
  if (devno >= 64 || !attr[devno][di]) {
    const int mx = (int)(es * (kTT + 1) * 32 * 33);
    SIGB_CUDA_TRY(di == 0 ? cudaFuncSetAttribute((const void*)jit_sample_grads<float>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, mx)
                          : cudaFuncSetAttribute((const void*)jit_sample_grads<double>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    if (devno < 64) attr[devno][di] = true;
  }
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t Bc = std::min(chunk, B - b0);
    const char* Xc = (const char*)X + es * (size_t)b0 * L * d;
    const char* Sc = (const char*)S + es * (size_t)b0 * s_ld;
    const char* gc = (const char*)g + es * (size_t)b0 * g_ld;
    long long Bl = Bc, Ll = L, sl = s_ld, s0 = s_col0, gl = g_ld, g0 = g_col0, Bp = pad32(Bc);
    void* Xv = (void*)Xc;
    void* Sv = (void*)Sc;
    void* gv = (void*)gc;
    int grp = groups, nblocks = (int)((Bc + 31) / 32), bulk = bulk_ok(Xc, dtype, d);
    if ((rc = zero_counters(ctr, groups, stream))) return rc;
    void* args[] = {&Xv, &Bl, &Ll, &Sv, &sl, &s0, &gv, &gl, &g0, &work, &Bp, &nblocks, &grp, &ctr, &bulk};
    const size_t smem = smem_bytes(dtype, (int)d, c, true);
    const void* kern = (const void*)p->jit.kern[di][1];
    count_launch(2);
    timing_begin(1, stream);
    const int threads = 32 * c.warps * c.pb;
    SIGB_CUDA_TRY(cudaLaunchKernel(
        kern, dim3(persistent_grid(kern, threads, smem, ((int64_t)groups * nblocks + c.pb - 1) / c.pb)), dim3(threads),
        args, smem, stream));
    timing_end(1, stream);
    const dim3 sgrid((unsigned)((L + kTT - 1) / kTT), (unsigned)((Bc + 31) / 32));
    const size_t ssm = es * (size_t)(kTT + 1) * d * 33;
    if (dtype == SIGB_F32)
      jit_sample_grads<float><<<sgrid, 256, ssm, stream>>>((const float*)work, Bp, Bc, groups, M, (int)d, b0,
                                                           (float*)dX, (float*)dinc);
    else
      jit_sample_grads<double><<<sgrid, 256, ssm, stream>>>((const double*)work, Bp, Bc, groups, M, (int)d, b0,
                                                            (double*)dX, (double*)dinc);
    SIGB_CUDA_TRY(cudaGetLastError());
  }
  return SIGB_OK;
}

}  // namespace jit
}  // namespace sigb

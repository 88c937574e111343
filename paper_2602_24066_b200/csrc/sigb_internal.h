// Internal definitions shared by the sigkit_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sigkit_b200.h"

namespace sigb {

// Longest word the device kernels schedule (level tables are fixed-size).
constexpr int kMaxLevel = 32;
// Steps of samples staged in shared memory per chunk.
constexpr int kChunk = 32;

// Records `msg` as the thread's last error and returns `code`.
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define SIGB_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::sigb::cuda_fail(_e, #expr); \
  } while (0)

// One independent part of the trie: a run of consecutive sibling subtrees
// plus the (replicated) chain of their common ancestors.  Local node order is
// canonical (level asc, code asc), so every level is a contiguous local range.
struct PartDesc {
  int n;         // local nodes (chain + subtrees)
  int node_off;  // offset into the node tables
  int tv_size;   // T-vector entries T(w, m), m > |w|
  int tb_size;   // adjoint entries Tbar(w, m), m >= |w|
  int lseg_off;  // offset into the letter-segment table (d + 1 entries)
  int depth;     // deepest level present
  int lvl[kMaxLevel + 2];  // lvl[l] = first local node of level l (1-based), lvl[depth+1] = n
};

// Node table entry A: {parent T-vector offset (-1: parent is the empty word),
//  letter | level << 8 | maxdesc << 16 | owner << 24, own T-vector offset (-1: none),
//  own adjoint offset}
// Node table entry B: {closure index, emitted index in I (-1: closure only),
//  first child (local), child count}.  Only the owner part emits / seeds a node.
struct PlanDev {
  const PartDesc* parts;
  const int4* nodeA;
  const int4* nodeB;
  const int* perm;  // per part: local ids sorted by (letter, id)
  const int* lseg;  // per part: d + 1 segment starts into perm
  int num_parts;
  int d;
  int max_len;
};

// Prefix closure cl(I) of a word set as a trie, canonical (length, code) order.
struct Trie {
  int64_t d = 0;
  int max_len = 0;
  std::vector<uint64_t> code;   // closure, canonical order
  std::vector<int64_t> len;
  std::vector<int64_t> parent;  // closure index, -1 for the empty word
  std::vector<int64_t> child_first, child_count;
  std::vector<int> md;          // deepest descendant length (incl. self)
  std::vector<int64_t> cost;    // subtree shared-memory cost (elements)
  std::vector<int64_t> emit;    // emitted index in I or -1
};

// Host image of a fragment plan (sigb_frag.cuh).  Per-fragment arrays are
// slot-major: [slot][Fp].
struct FragHost {
  int NC = 0, G = 0, K = 0;  // template shape
  int F = 0, cpp = 0, Fp = 0;
  double cost = 0;           // estimated issue slots per path-step (forward)
  std::vector<unsigned char> letter;  // [NGS][Fp], d = none
  std::vector<int> cidx, eidx, sidx;  // [NS][Fp]
  // backward gradient parking: slot (s, f) writes to pos[s][f] of a per-CTA
  // letter-major buffer; letter z of CTA-part c owns float4s [off[c][z], off[c][z+1])
  std::vector<unsigned short> pos;  // [NGS][Fp]
  std::vector<int> red_off;         // [cpp][d+1] in float4 units
  int pstride = 0;                  // floats per parked step (4-aligned, + trash)
};

// Builds the fragment decomposition of `t` for the best available template
// shape; false (with `why`) when no instantiation fits.
bool plan_fragments(const Trie& t, FragHost& out, std::string& why);

// Word-set-specialised (NVRTC) kernels for small tries (sigb_jit.cu).
namespace jit {
struct Task {
  std::vector<int64_t> nodes;  // closure indices: chain (levels 1..c) then bodies, topological
  int chain = 0;               // leading chain nodes (replicated; the first task containing one owns it)
};
// Launch shape of one generated kernel: warps (= tasks) per slot, slots (path
// blocks) per CTA, steps per staged chunk, minimum resident CTAs per SM
// (register budget), T-node cap per task.
struct Cfg {
  int warps = 4, ch = 8, minb = 4, pb = 1;
  int lock = 0;  // slots claim together and share the CTA barrier (lockstep)
  int maxreg = 0;  // NVRTC --maxrregcount (0: launch bounds only)
  int64_t cap = 96;
};
struct Pending;  // a background NVRTC compile (sigb_jit.cu)
}  // namespace jit
struct JitHost {
  std::vector<jit::Task> fwd_tasks, bwd_tasks;
  jit::Cfg cfg[2][2];  // [dtype f32=0/f64=1][backward]
};
struct JitPlan {
  bool eligible = false;       // small enough for generated code
  Trie trie;                   // closure (kept for lazy code generation)
  JitHost host;
  // compiled kernels per [dtype][backward]; failed = compile attempted and failed
  void* lib[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  void* kern[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  bool failed[2][2] = {{false, false}, {false, false}};
  bool broken = false;  // some compilation failed: route this plan elsewhere
  // the fragment kernels served a call while the cubin compiled: this plan keeps serving that
  // [dtype][direction] with them, so its results stay bitwise reproducible call to call (the
  // reference's determinism contract); the cubin lands in the cache for later plans / processes
  bool standin[2][2] = {{false, false}, {false, false}};
  std::shared_ptr<jit::Pending> pending[2][2];  // background compiles in flight / finished
  std::mutex mu;                                // guards the compile / load state above
};
namespace jit {
bool eligible(const Trie& t);
void make_plan(const Trie& t, JitHost& h);
std::string source(const Trie& t, const JitHost& h, int dtype, bool backward);
// Compile / load the generated kernel.  A cubin-cache hit loads at once; otherwise,
// unless `wait`, the NVRTC compile runs on a background host thread and ensure
// returns kPending (the caller serves the call with the fragment kernels) -- from then
// on for this plan, dtype and direction (JitPlan::standin).  SIGB_OK when the kernel is
// loaded, else an error code.
constexpr int kPending = -1;
int ensure(sigb_plan* p, int dtype, bool backward, bool wait);
bool wait_default();  // policy 4 or SIGB_JIT_SYNC=1: compile synchronously
int precompile(const Trie& t, int dtype, bool backward);  // host-only: fill the cubin cache
int forward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, void* out, int64_t out_ld,
            int64_t out_col0, int include_empty, void* state, cudaStream_t stream);
size_t backward_workspace(const sigb_plan* p, int dtype, int64_t B, int64_t L);
int backward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream);
}  // namespace jit

struct FragDevPlan {
  bool ok = false;
  int NC = 0, G = 0, K = 0, F = 0, cpp = 0, Fp = 0, pstride = 0;
  unsigned char* letter = nullptr;
  int *cidx = nullptr, *eidx = nullptr, *sidx = nullptr;
  unsigned short* pos = nullptr;
  int* red_off = nullptr;
};

}  // namespace sigb

struct sigb_plan {
  int device = 0;  // CUDA device current at sigb_plan_create; entry points switch to it (DeviceGuard)
  int64_t d = 0;
  int64_t W = 0;   // emitted words |I|
  int64_t Wc = 0;  // closure |cl(I)|
  int max_len = 0;
  bool prefix_closed = true;
  int trunc_depth = 0;  // N when cl(I) is the full truncation of depth N, else 0
  int num_parts = 0;
  int64_t step_fmas = 0;
  // per-dtype-agnostic smem requirements (in elements of the compute type)
  int max_n = 0, max_tv = 0, max_tb = 0;
  // device arrays
  sigb::PartDesc* d_parts = nullptr;
  int4* d_nodeA = nullptr;
  int4* d_nodeB = nullptr;
  int* d_perm = nullptr;
  int* d_lseg = nullptr;
  std::vector<sigb::PartDesc> h_parts;
  sigb::FragDevPlan frag;  // register-resident fragment kernels (sigb_frag.cuh), when ok
  sigb::JitPlan jit;       // word-set-specialised kernels (sigb_jit.cu), when eligible

  sigb::PlanDev dev() const {
    sigb::PlanDev p;
    p.parts = d_parts;
    p.nodeA = d_nodeA;
    p.nodeB = d_nodeB;
    p.perm = d_perm;
    p.lseg = d_lseg;
    p.num_parts = num_parts;
    p.d = (int)d;
    p.max_len = max_len;
    return p;
  }
};

namespace sigb {
// Makes `dev` current for the scope and restores the caller's device: every C-ABI call
// taking a plan launches on the plan's device whatever the calling thread has current.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
// kernel-routing policy (sigb_set_kernel_policy), tensor-core switch (sigb_set_tensor_cores)
// and launch counter
extern int g_policy;
extern int g_tensor_cores;
// per-process byte budget for a backward's per-chunk workspace (partials, checkpoints)
size_t partial_budget();
void count_launch(int n = 1);
// Optional CUDA-event timing of the main kernels (sigb_timing_enable):
// `which` 0 = forward Chen kernel, 1 = backward Chen kernel (summed over batch chunks).
void timing_begin(int which, cudaStream_t stream);
void timing_end(int which, cudaStream_t stream);
namespace frag {
bool supported(int NC, int G, int K);
// bounds (K, 2) / K: windowed forward over B*K virtual paths (bounds NULL, K 1: whole paths)
int forward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, const int64_t* bounds, int64_t K,
            void* out, int64_t out_ld, int64_t out_col0, int include_empty, void* state, cudaStream_t stream);
// stride > 0: checkpoint_stride (replay + reload, frag_ckpt_kernel); the workspace adds the rows
size_t backward_workspace(const sigb_plan* p, int dtype, int64_t B, int64_t L, int64_t stride = 0);
int backward(const sigb_plan* p, int dtype, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream, int64_t stride = 0);
}  // namespace frag
namespace trunc {
bool supported(int64_t d, int depth);
int64_t forward_ctas(int64_t d, int depth, int64_t B);  // grid of the truncated forward for B paths
int forward(int dtype, int64_t d, int depth, const void* X, int64_t B, int64_t L, const int64_t* bounds, int64_t K,
            void* out, int64_t out_ld, int64_t out_col0, int include_empty, cudaStream_t stream);
// stride > 0: the reference's checkpoint_stride (backward.py:183-199): a forward replay stores the
// prefix levels every `stride` steps and the reverse sweep reloads them there
size_t backward_workspace(int dtype, int64_t d, int depth, int64_t B, int64_t L, int64_t stride = 0);
int backward(int dtype, int64_t d, int depth, const void* X, int64_t B, int64_t L, const void* S, int64_t s_ld,
             int64_t s_col0, const void* g, int64_t g_ld, int64_t g_col0, void* work, size_t work_bytes, void* dX,
             void* dinc, cudaStream_t stream, int64_t stride = 0);
}  // namespace trunc
int launch_wordset_tables(const uint64_t* d_codes, const int64_t* d_lengths, int64_t W, int64_t d,
                          int64_t max_len, int64_t* d_letters, int64_t* d_prefix, int64_t* d_suffix,
                          int64_t* d_level_start, uint64_t* d_packed, cudaStream_t stream);
}  // namespace sigb

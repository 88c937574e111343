// Fragment planner: cuts the prefix closure cl(I) into the per-thread
// fragments of sigb_frag.cuh (host code, runs once per word set).
//
// Node classes of the trie:
//   leaf         no children;
//   leaf-parent  internal, every child is a leaf ("mid" of a fragment);
//   anchor       the empty word and every other internal node.
// A fragment = (anchor a, its ancestor chain, <= G leaf-parent children of a
// with <= K leaf letters each from one shared list LL, <= K leaf children of a).
// Every closure node lands in exactly one fragment as its OWNER (emits it,
// seeds its adjoint); chain ancestors are replicated read-only elsewhere.
// The reference needs no such cut (one numba unit per (path, word),
// _kernels.py:46-58); here it is what lets the state live in registers.
#include <algorithm>
#include <map>

#include "sigb_internal.h"

namespace sigb {
namespace {

struct Piece {
  int64_t mid;                  // closure index of the leaf-parent
  std::vector<int> letters;     // leaf letters carried by this piece (sorted)
  std::vector<int64_t> leaves;  // matching leaf closure indices
  bool owner;                   // emits the mid itself
};

struct Frag {
  int64_t anchor;  // closure index, -1 for the empty word
  int la;          // anchor level
  std::vector<Piece> mids;
  std::vector<int> al;          // anchor-leaf letters
  std::vector<int64_t> al_node;
};

int letter_of(const Trie& t, int64_t i) { return (int)(t.code[i] % (uint64_t)t.d); }

std::vector<int> merged(const std::vector<int>& a, const std::vector<int>& b) {
  std::vector<int> u;
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(u));
  return u;
}

// Greedy cut for one (G, K).
std::vector<Frag> cut(const Trie& t, int G, int K) {
  const int64_t Wc = (int64_t)t.code.size();
  auto is_leaf = [&](int64_t i) { return t.child_count[i] == 0; };
  auto is_lp = [&](int64_t i) {
    if (is_leaf(i)) return false;
    for (int64_t c = t.child_first[i]; c < t.child_first[i] + t.child_count[i]; ++c)
      if (!is_leaf(c)) return false;
    return true;
  };
  // children of the empty word: the level-1 block
  int64_t n1 = 0;
  while (n1 < Wc && t.len[n1] == 1) ++n1;
  std::vector<Frag> frags;
  auto process = [&](int64_t a, int64_t cf, int64_t cc) {
    std::vector<Piece> pieces;
    std::vector<int> al;
    std::vector<int64_t> al_node;
    for (int64_t c = cf; c < cf + cc; ++c) {
      if (is_leaf(c)) {
        al.push_back(letter_of(t, c));
        al_node.push_back(c);
      } else if (is_lp(c)) {
        std::vector<int> lets;
        std::vector<int64_t> nodes;
        for (int64_t x = t.child_first[c]; x < t.child_first[c] + t.child_count[c]; ++x) {
          lets.push_back(letter_of(t, x));
          nodes.push_back(x);
        }
        for (size_t s = 0; s < lets.size(); s += (size_t)K) {
          size_t e = std::min(lets.size(), s + (size_t)K);
          pieces.push_back(Piece{c, std::vector<int>(lets.begin() + s, lets.begin() + e),
                                 std::vector<int64_t>(nodes.begin() + s, nodes.begin() + e), s == 0});
        }
      }
    }
    if (pieces.empty() && al.empty()) return;
    std::stable_sort(pieces.begin(), pieces.end(),
                     [](const Piece& x, const Piece& y) { return x.letters < y.letters; });
    const int la = a < 0 ? 0 : (int)t.len[a];
    std::vector<Frag> mine;
    std::vector<std::vector<int>> unions;
    for (Piece& p : pieces) {
      bool placed = false;
      if (!mine.empty() && (int)mine.back().mids.size() < G) {
        std::vector<int> u = merged(unions.back(), p.letters);
        if ((int)u.size() <= K) {
          mine.back().mids.push_back(p);
          unions.back() = u;
          placed = true;
        }
      }
      if (!placed) {
        mine.push_back(Frag{a, la, {p}, {}, {}});
        unions.push_back(p.letters);
      }
    }
    for (size_t s = 0, i = 0; s < al.size(); s += (size_t)K, ++i) {
      if (i == mine.size()) mine.push_back(Frag{a, la, {}, {}, {}});
      size_t e = std::min(al.size(), s + (size_t)K);
      mine[i].al.assign(al.begin() + s, al.begin() + e);
      mine[i].al_node.assign(al_node.begin() + s, al_node.begin() + e);
    }
    for (Frag& f : mine) frags.push_back(std::move(f));
  };
  process(-1, 0, n1);
  for (int64_t a = 0; a < Wc; ++a)
    if (!is_leaf(a) && !is_lp(a)) process(a, t.child_first[a], t.child_count[a]);
  return frags;
}

// Issue slots of one fragment-step of the forward (FP + LDS), the planner's cost model.
double frag_cost(int NC, int G, int K) {
  const int NV = NC + 2;
  double c = 0;
  for (int k = 0; k < NC; ++k) c += 2.0 * (NV - k) - 1;  // FMA per target + FMUL per r > 1
  c += NC + G + 2.0 * K;                                  // increment gathers
  c += 3.0 * G + (double)G * K + K;                       // mids, leaves, anchor leaves
  return c;
}

struct Shape3 {
  int G, K;
};
// (G, K) shapes instantiated in sigb_frag.cu (NC = 1..5 each).
const Shape3 kShapes[] = {{5, 5}, {4, 4}, {2, 8}, {1, 16}};
constexpr int kMaxNC = 5;

}  // namespace

bool plan_fragments(const Trie& t, FragHost& out, std::string& why) {
  const int64_t Wc = (int64_t)t.code.size();
  if (t.d > 254) {
    why = "fragment kernels need d <= 254";
    return false;
  }
  double best = -1;
  std::vector<Frag> best_frags;
  int bestG = 0, bestK = 0, bestNC = 0;
  for (const Shape3& sh : kShapes) {
    std::vector<Frag> fr = cut(t, sh.G, sh.K);
    int NC = 1;
    for (const Frag& f : fr) NC = std::max(NC, f.la);
    if (NC > kMaxNC || fr.empty()) continue;
    const double c = (double)fr.size() * frag_cost(NC, sh.G, sh.K);
    if (best < 0 || c < best) {
      best = c;
      best_frags = std::move(fr);
      bestG = sh.G;
      bestK = sh.K;
      bestNC = NC;
    }
  }
  if (best < 0) {
    why = "no fragment shape fits (anchor deeper than " + std::to_string(kMaxNC) + ")";
    return false;
  }
  const int NC = bestNC, G = bestG, K = bestK;
  const int NS = NC + G + G * K + K, NGS = NC + G + 2 * K;
  const int F = (int)best_frags.size();
  const int TPB = 128;
  const int cpp = (F + TPB - 1) / TPB;
  const int Fp = cpp * TPB;
  const unsigned char none = (unsigned char)t.d;
  out = FragHost();
  out.NC = NC;
  out.G = G;
  out.K = K;
  out.F = F;
  out.cpp = cpp;
  out.Fp = Fp;
  out.cost = best;
  out.letter.assign((size_t)NGS * Fp, none);
  out.cidx.assign((size_t)NS * Fp, -1);
  out.eidx.assign((size_t)NS * Fp, -1);
  out.sidx.assign((size_t)NS * Fp, -1);
  std::vector<char> owned(Wc, 0);
  auto own = [&](int slot, int f, int64_t node) {
    if (owned[node]) return;
    owned[node] = 1;
    out.eidx[(size_t)slot * Fp + f] = (int)t.emit[node];
    out.sidx[(size_t)slot * Fp + f] = (int)node;
  };
  for (int f = 0; f < F; ++f) {
    const Frag& fr = best_frags[f];
    // chain: identity padding, then ancestors level 1..la (the anchor last)
    std::vector<int64_t> chain;
    for (int64_t u = fr.anchor; u >= 0; u = t.parent[u]) chain.push_back(u);
    std::reverse(chain.begin(), chain.end());
    const int off = NC - (int)chain.size();
    for (int k = 0; k < NC; ++k) {
      if (k < off) {
        out.cidx[(size_t)k * Fp + f] = -2;  // identity node: S = 1, increment 0
        continue;
      }
      const int64_t u = chain[k - off];
      out.letter[(size_t)k * Fp + f] = (unsigned char)letter_of(t, u);
      out.cidx[(size_t)k * Fp + f] = (int)u;
      own(k, f, u);
    }
    // shared leaf-letter list
    std::vector<int> LL;
    for (const Piece& p : fr.mids) LL = merged(LL, p.letters);
    for (int k = 0; k < (int)LL.size(); ++k) out.letter[(size_t)(NC + G + k) * Fp + f] = (unsigned char)LL[k];
    for (int g = 0; g < (int)fr.mids.size(); ++g) {
      const Piece& p = fr.mids[g];
      out.letter[(size_t)(NC + g) * Fp + f] = (unsigned char)letter_of(t, p.mid);
      out.cidx[(size_t)(NC + g) * Fp + f] = (int)p.mid;
      if (p.owner) own(NC + g, f, p.mid);
      for (size_t i = 0; i < p.letters.size(); ++i) {
        const int k = (int)(std::lower_bound(LL.begin(), LL.end(), p.letters[i]) - LL.begin());
        const int slot = NC + G + g * K + k;
        out.cidx[(size_t)slot * Fp + f] = (int)p.leaves[i];
        own(slot, f, p.leaves[i]);
      }
    }
    for (int k = 0; k < (int)fr.al.size(); ++k) {
      out.letter[(size_t)(NC + G + K + k) * Fp + f] = (unsigned char)fr.al[k];
      const int slot = NC + G + G * K + k;
      out.cidx[(size_t)slot * Fp + f] = (int)fr.al_node[k];
      own(slot, f, fr.al_node[k]);
    }
  }
  for (int64_t i = 0; i < Wc; ++i)
    if (!owned[i]) {
      why = "internal: fragment cut missed closure node " + std::to_string(i);
      return false;
    }
  // per CTA-part letter-major parking layout for the backward's gradient terms:
  // letter z's entries are contiguous (slot-major, then thread), each letter
  // block padded to a float4; slots without a letter (0xFFFF) are not parked.
  out.pos.assign((size_t)NGS * Fp, 0);
  out.red_off.assign((size_t)cpp * (t.d + 1), 0);
  int pmax = 0;
  for (int c = 0; c < cpp; ++c) {
    std::vector<int> cnt(t.d, 0);
    for (int slot = 0; slot < NGS; ++slot)
      for (int tid = 0; tid < TPB; ++tid) {
        const int z = out.letter[(size_t)slot * Fp + c * TPB + tid];
        if (z < t.d) cnt[z]++;
      }
    std::vector<int> base(t.d + 1, 0);
    for (int z = 0; z < t.d; ++z) base[z + 1] = base[z] + (cnt[z] + 3) / 4 * 4;
    for (int z = 0; z <= t.d; ++z) out.red_off[(size_t)c * (t.d + 1) + z] = base[z] / 4;
    std::vector<int> fill(base.begin(), base.end() - 1);
    for (int slot = 0; slot < NGS; ++slot)
      for (int tid = 0; tid < TPB; ++tid) {
        const size_t i = (size_t)slot * Fp + c * TPB + tid;
        const int z = out.letter[i];
        out.pos[i] = (unsigned short)(z < t.d ? fill[z]++ : 0xFFFF);  // no letter: not parked
      }
    pmax = std::max(pmax, base[t.d]);
  }
  if (pmax >= 65535) {
    why = "fragment gradient buffer exceeds 16-bit offsets";
    return false;
  }
  out.pstride = pmax;
  return true;
}

}  // namespace sigb

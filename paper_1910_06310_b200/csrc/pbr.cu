// K2: device partition-based reordering (pbr_reorder, reorder.py:361-404),
// bit-exact with the reference.
//
// One CTA per graph.  The algorithm is inherently a sequence of greedy moves,
// so the CTA parallelises each move's gain evaluation and first-max argmax
// (block reductions over packed (gain, -index) keys) and applies the move's
// integer bookkeeping with atomics (integer adds commute, so the state is
// exact regardless of order).  Restated semantics:
//   * adjacency = sorted unique neighbours, expanded from the device octiles;
//   * two candidates (natural order, SplitMix64(seed) Fisher-Yates shuffle,
//     rng.py:31-62), each: recursive balanced bisection (2-way FM on the edge
//     cut, reorder.py:282-352) then K-way FM on the connected-part-pair
//     objective with the reference's literal gain formula, including the
//     saturating boolean 'appear' term (reorder.py:171-274);
//   * natural wins ties; permutation ranks nodes by (part, id);
//   * identity fallbacks on the pair objective and on the octile count.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/mgk.h"
#include "mgk_internal.h"
#include "pbr.h"

namespace mgk {

constexpr int kPbrThreads = 512;
constexpr int kPbrWarps = kPbrThreads / 32;
constexpr int kMaxPasses = 10;
constexpr int kLogMax = 512;
__device__ int g_pbr_log[1 + 4 * kLogMax];  // debug: first FM moves of block 0 (u, dst, gain, pass)
// profile: SM cycles of the slowest graph's phases (max over graphs): bisection, K-way FM, rest
__device__ unsigned long long g_pbr_cycles[3];

struct PbrScratch {
  int* rowptr;   // n + 1
  int* adj;      // S (sorted unique neighbours)
  int* parts;    // n   current partition
  int* cand;     // 2n  candidate partitions
  int* order;    // n   recursion node order
  int* tmp;      // n
  int* posmap;   // n   global -> local position (-1 outside the bisect task)
  int* side;     // n
  int* conn2;    // 2n  bisect: neighbours on side 0 / 1
  int* locked;   // n
  int* hist;     // 4n  (node, src); forced moves can relocate locked nodes, so up to 2n moves
  int* conn;     // n*k
  int* ec;       // k*k
  int* sizes;    // k
  int* targets;  // k
  unsigned* adjbits;  // k x W   bit Q of row P: ec[P][Q] > 0 (P != Q), W = ceil(k / 32)
  unsigned* elig;     // W       destination parts allowed for the current move
  unsigned long long* kcache;  // n   balanced-state best-move key of every node (FM key cache)
  int* kvalid;        // n       cache entry still exact
  unsigned* pmask;    // W       parts touched by the last move (cache invalidation)
  unsigned* fmask;    // W       parts whose adjacency-bit row flipped during the last move
  int* npl;           // S       per node: the distinct parts of its neighbours (capacity = degree,
                      //         laid out like adj), maintained incrementally by every move
  int* npc;           // n       their count
  int* flip;          // 1       an adjacency bit flipped during the last move
  int* stack;    // 6k   recursion tasks (begin, end, first_part, nparts)
  int* dbg;      // 2n   candidates before FM refinement (parity triage)
};

__host__ __device__ inline int pbr_words(int k) { return (k + 31) >> 5; }

__host__ __device__ inline int64_t pbr_scratch_ints(int n, int S, int k) {
  return (int64_t)(n + 1) + S + n + 2 * n + n + n + n + n + 2 * n + n + 4 * n + (int64_t)n * k + (int64_t)k * k + k +
         k + (int64_t)k * pbr_words(k) + pbr_words(k) + (2 * (int64_t)n + 2) + n + 2 * pbr_words(k) + 1 + S + n +
         6 * (int64_t)k + 2 * (int64_t)n + 64;
}

__device__ PbrScratch carve(int* base, int n, int S, int k) {
  PbrScratch s;
  int* p = base;
  s.rowptr = p; p += n + 1;
  s.adj = p; p += S;
  s.parts = p; p += n;
  s.cand = p; p += 2 * n;
  s.order = p; p += n;
  s.tmp = p; p += n;
  s.posmap = p; p += n;
  s.side = p; p += n;
  s.conn2 = p; p += 2 * n;
  s.locked = p; p += n;
  s.hist = p; p += 4 * n;
  s.conn = p; p += (int64_t)n * k;
  s.ec = p; p += (int64_t)k * k;
  s.sizes = p; p += k;
  s.targets = p; p += k;
  s.adjbits = reinterpret_cast<unsigned*>(p); p += (int64_t)k * pbr_words(k);
  s.elig = reinterpret_cast<unsigned*>(p); p += pbr_words(k);
  if ((p - base) & 1) ++p;  // 8-byte alignment of the key cache
  s.kcache = reinterpret_cast<unsigned long long*>(p); p += 2 * (int64_t)n;
  s.kvalid = p; p += n;
  s.pmask = reinterpret_cast<unsigned*>(p); p += pbr_words(k);
  s.fmask = reinterpret_cast<unsigned*>(p); p += pbr_words(k);
  s.flip = p; p += 1;
  s.npl = p; p += S;
  s.npc = p; p += n;
  s.stack = p;
  p += 6 * k;
  s.dbg = p;
  return s;
}

// ---- block reductions ------------------------------------------------------
__device__ unsigned long long block_max_u64(unsigned long long v, unsigned long long* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long m = red[0];
  for (int w = 1; w < kPbrWarps; ++w) m = red[w] > m ? red[w] : m;
  return m;
}

__device__ long long block_sum_i64(long long v, long long* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long m = 0;
  for (int w = 0; w < kPbrWarps; ++w) m += red[w];
  return m;
}

// exclusive scan of flags over [0, n) in chunks; returns the total
__device__ int block_stable_positions(const int* flag, int* out, int n, int* shw, int* shc) {
  if (threadIdx.x == 0) *shc = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int f = (i < n) ? flag[i] : 0;
    const unsigned b = __ballot_sync(0xffffffffu, f);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int within = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) shw[w] = __popc(b);
    __syncthreads();
    int before = *shc;
    for (int k = 0; k < w; ++k) before += shw[k];
    if (i < n) out[i] = before + within;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int k = 0; k < kPbrWarps; ++k) tot += shw[k];
      *shc += tot;
    }
    __syncthreads();
  }
  return *shc;
}

// ---- SplitMix64 (rng.py:31-62) ---------------------------------------------
struct SplitMix64 {
  uint64_t s;
  __device__ uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ uint64_t randint(uint64_t n) {  // rejection: z < 2^64 - (2^64 mod n)
    const uint64_t rem = (0ull - n) % n;
    for (;;) {
      const uint64_t z = next();
      if (rem == 0 || z < 0ull - rem) return z % n;
    }
  }
};

// ---- recursive bisection (reorder.py:282-352) --------------------------------
// 2-way FM on the nodes order[b, e) with cap nodes on side 0; stable partition.
__device__ void bisect(PbrScratch& s, int b, int e, int cap, unsigned long long* red64, long long* redll, int* shw,
                       int* shc, int* shi) {
  const int nt = e - b;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    s.posmap[s.order[b + i]] = i;
    s.side[i] = i < cap ? 0 : 1;
    s.locked[i] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int u = s.order[b + i];
    int c0 = 0, c1 = 0;
    for (int q = s.rowptr[u]; q < s.rowptr[u + 1]; ++q) {
      const int j = s.posmap[s.adj[q]];
      if (j >= 0) (s.side[j] ? c1 : c0)++;
    }
    s.conn2[2 * i] = c0;
    s.conn2[2 * i + 1] = c1;
  }
  __syncthreads();
  const int t0 = cap, t1 = nt - cap;
  for (int pass = 0; pass < kMaxPasses; ++pass) {
    long long cutl = 0, sz0l = 0;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      cutl += s.conn2[2 * i + 1 - s.side[i]];
      sz0l += s.side[i] == 0;
      s.locked[i] = 0;
    }
    long long cut = block_sum_i64(cutl, redll) / 2;
    int size0 = (int)block_sum_i64(sz0l, redll);
    int size1 = nt - size0;
    long long cur = cut, best = cut;
    int prefix = 0, hlen = 0;
    for (;;) {
      const bool bal = (size0 == t0 && size1 == t1);
      const int over = bal ? -1 : (size0 > t0 ? 0 : 1);
      unsigned long long key = 0;
      for (int i = threadIdx.x; i < nt; i += blockDim.x) {
        if (s.locked[i] || (!bal && s.side[i] != over)) continue;
        const int sd = s.side[i];
        const long long g = (long long)s.conn2[2 * i + 1 - sd] - s.conn2[2 * i + sd];
        // max gain, then lowest position (reorder.py:315-316 first argmax)
        const unsigned long long k = ((unsigned long long)(g + (1ll << 30)) << 32) | (0xFFFFFFFFu - (unsigned)i);
        key = k > key ? k : key;
      }
      key = block_max_u64(key, red64);
      if (key == 0) break;
      const int pick = (int)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFu));
      const long long g = (long long)(key >> 32) - (1ll << 30);
      const int sd = s.side[pick];
      __syncthreads();
      // flip pick; neighbours' side counts move
      const int u = s.order[b + pick];
      for (int q = s.rowptr[u] + threadIdx.x; q < s.rowptr[u + 1]; q += blockDim.x) {
        const int j = s.posmap[s.adj[q]];
        if (j >= 0) {
          atomicSub(&s.conn2[2 * j + sd], 1);
          atomicAdd(&s.conn2[2 * j + 1 - sd], 1);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        s.side[pick] = 1 - sd;
        s.locked[pick] = 1;
        s.hist[hlen] = pick;
      }
      cur -= g;
      ++hlen;
      if (sd == 0) { --size0; ++size1; } else { ++size0; --size1; }
      if (size0 == t0 && size1 == t1 && cur < best) {
        best = cur;
        prefix = hlen;
      }
      __syncthreads();
    }
    // roll back history[prefix:] in reverse
    for (int h = hlen - 1; h >= prefix; --h) {
      const int i = s.hist[h];
      const int sd = s.side[i];
      const int u = s.order[b + i];
      for (int q = s.rowptr[u] + threadIdx.x; q < s.rowptr[u + 1]; q += blockDim.x) {
        const int j = s.posmap[s.adj[q]];
        if (j >= 0) {
          atomicSub(&s.conn2[2 * j + sd], 1);
          atomicAdd(&s.conn2[2 * j + 1 - sd], 1);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) s.side[i] = 1 - sd;
      __syncthreads();
    }
    if (prefix == 0) break;
  }
  // stable partition: left = side 0 in order, right = side 1 in order
  for (int i = threadIdx.x; i < nt; i += blockDim.x) s.locked[i] = (s.side[i] == 0);
  __syncthreads();
  const int nleft = block_stable_positions(s.locked, s.conn2, nt, shw, shc);
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int dst = s.side[i] == 0 ? s.conn2[i] : nleft + (i - s.conn2[i]);
    s.tmp[dst] = s.order[b + i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    s.order[b + i] = s.tmp[i];
    s.posmap[s.tmp[i]] = -1;
  }
  __syncthreads();
  (void)shi;
}

// _recursive_parts (reorder.py:344-352) with an explicit task stack
__device__ void recursive_parts(PbrScratch& s, int n, int k, int* outparts, unsigned long long* red64, long long* redll,
                                int* shw, int* shc, int* shi) {
  auto part_size = [&](int p) { return p < k - 1 ? kTile : n - kTile * (k - 1); };
  __shared__ int sp;
  if (threadIdx.x == 0) {
    sp = 0;
    s.stack[0] = 0;
    s.stack[1] = n;
    s.stack[2] = 0;
    s.stack[3] = k;
    sp = 1;
  }
  __syncthreads();
  while (sp > 0) {
    const int top = sp - 1;
    const int b = s.stack[4 * top], e = s.stack[4 * top + 1], first = s.stack[4 * top + 2], np = s.stack[4 * top + 3];
    __syncthreads();
    if (threadIdx.x == 0) sp = top;
    __syncthreads();
    if (np == 1) {
      for (int i = b + threadIdx.x; i < e; i += blockDim.x) outparts[s.order[i]] = first;
      __syncthreads();
      continue;
    }
    const int kl = (np + 1) / 2;
    int cap = 0;
    for (int p = first; p < first + kl; ++p) cap += part_size(p);
    bisect(s, b, e, cap, red64, redll, shw, shc, shi);
    if (threadIdx.x == 0) {
      // push right then left so the left task runs first (order is irrelevant to the result)
      int t = sp;
      s.stack[4 * t] = b + cap;
      s.stack[4 * t + 1] = e;
      s.stack[4 * t + 2] = first + kl;
      s.stack[4 * t + 3] = np - kl;
      ++t;
      s.stack[4 * t] = b;
      s.stack[4 * t + 1] = b + cap;
      s.stack[4 * t + 2] = first;
      s.stack[4 * t + 3] = kl;
      sp = t + 1;
    }
    __syncthreads();
  }
}

// ---- K-way FM (reorder.py:171-274) ---------------------------------------------
__device__ long long ec_objective(const PbrScratch& s, int k, long long* redll) {
  long long c = 0;
  for (int64_t x = threadIdx.x; x < (int64_t)k * k; x += blockDim.x) {
    const int P = (int)(x / k), Q = (int)(x - (int64_t)P * k);
    c += (P < Q && s.ec[x] > 0);
  }
  return block_sum_i64(c, redll);
}

// adjacency bit (P, Q) <- ec[P][Q] > 0 (diagonal never stored; it never enters a gain)
__device__ __forceinline__ bool sync_adjbit(const PbrScratch& s, int k, int P, int Q) {
  if (P == Q) return false;
  const unsigned bit = 1u << (Q & 31);
  unsigned* wp = s.adjbits + (int64_t)P * pbr_words(k) + (Q >> 5);
  if (s.ec[(int64_t)P * k + Q] > 0) return !(atomicOr(wp, bit) & bit);
  return (atomicAnd(wp, ~bit) & bit) != 0;
}

__device__ __forceinline__ void mark_part(const PbrScratch& s, int P) { atomicOr(&s.pmask[P >> 5], 1u << (P & 31)); }
__device__ __forceinline__ void mark_flip(const PbrScratch& s, int P) {
  atomicOr(&s.fmask[P >> 5], 1u << (P & 31));
  *s.flip = 1;
}

__device__ void fm_move(PbrScratch& s, int k, int u, int dst) {
  const int src = s.parts[u];
  for (int q = s.rowptr[u] + threadIdx.x; q < s.rowptr[u + 1]; q += blockDim.x) {
    const int v = s.adj[q];
    const int p = s.parts[v];
    atomicSub(&s.ec[(int64_t)src * k + p], 1);
    atomicSub(&s.ec[(int64_t)p * k + src], 1);
    atomicAdd(&s.ec[(int64_t)dst * k + p], 1);
    atomicAdd(&s.ec[(int64_t)p * k + dst], 1);
    const int was_src = atomicSub(&s.conn[(int64_t)v * k + src], 1);
    const int was_dst = atomicAdd(&s.conn[(int64_t)v * k + dst], 1);
    // v's neighbour-part set: src leaves when its last link goes, dst joins with the first
    // (each v occurs once in u's adjacency, so one thread owns v's list here)
    int* l = s.npl + s.rowptr[v];
    if (was_src == 1) {
      const int c = s.npc[v];
      for (int t = 0; t < c; ++t)
        if (l[t] == src) {
          l[t] = l[c - 1];
          break;
        }
      s.npc[v] = c - 1;
    }
    if (was_dst == 0) l[s.npc[v]++] = dst;
  }
  __syncthreads();
  for (int q = s.rowptr[u] + threadIdx.x; q < s.rowptr[u + 1]; q += blockDim.x) {
    const int v = s.adj[q];
    const int p = s.parts[v];
    if (sync_adjbit(s, k, src, p)) mark_flip(s, src);
    if (sync_adjbit(s, k, p, src)) mark_flip(s, p);
    if (sync_adjbit(s, k, dst, p)) mark_flip(s, dst);
    if (sync_adjbit(s, k, p, dst)) mark_flip(s, p);
    // key-cache invalidation: v's conn row and neighbour parts changed; part p's ec row changed
    s.kvalid[v] = 0;
    mark_part(s, p);
  }
  if (threadIdx.x == 0) {
    s.kvalid[u] = 0;
    mark_part(s, src);
    mark_part(s, dst);
  }
  __syncthreads();
  if (threadIdx.x == 0) s.parts[u] = dst;
  __syncthreads();
}

// Drop the cached keys the last move may have changed: nodes of marked parts (their part's ec row
// changed) and, for every part whose adjacency-bit row flipped, the neighbours of its members (the
// nodes with that part in NP).  Clears the marks.
__device__ void invalidate_marked(PbrScratch& s, int n, int k) {
  const bool any_flip = *s.flip != 0;
  for (int w = threadIdx.x; w < n; w += blockDim.x) {
    const int P = s.parts[w];
    if ((s.pmask[P >> 5] >> (P & 31)) & 1u) s.kvalid[w] = 0;
    if (any_flip && ((s.fmask[P >> 5] >> (P & 31)) & 1u))
      for (int q = s.rowptr[w]; q < s.rowptr[w + 1]; ++q) s.kvalid[s.adj[q]] = 0;
  }
  __syncthreads();
  for (int w = threadIdx.x; w < pbr_words(k); w += blockDim.x) {
    s.pmask[w] = 0;
    s.fmask[w] = 0;
  }
  if (threadIdx.x == 0) *s.flip = 0;
  __syncthreads();
}

// Best move of node u under the reference's literal gain (reorder.py:171-189),
// as a packed first-max key (0: no allowed destination).  Restated so that the
// k destinations need not be scanned one by one:
//   NP = parts holding a neighbour of u (may include A = part(u)),
//   L  = sum_{P in NP, P != A} [ec[A][P] == conn[u][P]]        (the lose sum)
//   B in NP \ {A}: the formula term by term, with the saturating OR
//       appear = OR_{P in NP, P != B} [ec[B][P] == 0] - [pos A and ec[B][A] == 0];
//   B not in NP, B != A: conn[u][B] = 0 collapses the formula to
//       gain = L - OR_{P in NP} [ec[B][P] == 0]
//     (posA, ec[A][B] > 0: dab = 0, appear = OR;  posA, ec[A][B] = 0: dab = -1 and
//      the OR is 1 through P = A, appear = 0;  not posA: dab = 0, appear = OR),
//     so the best such B is the lowest allowed part adjacent to every part of NP
//     (gain L), else the lowest allowed part outside NP (gain L - 1).
// Ties keep the lowest B, as the flat row-major argmax does.
__device__ unsigned long long fm_node_key(const PbrScratch& s, int k, int u) {
  const int W = pbr_words(k);
  const int A = s.parts[u];
  const int* cu = s.conn + (int64_t)u * k;
  const int* ecA = s.ec + (int64_t)A * k;
  const int* np = s.npl + s.rowptr[u];  // distinct neighbour parts (order irrelevant below)
  const int nnp = s.npc[u];
  int L = 0;
  for (int t = 0; t < nnp; ++t) {
    const int P = np[t];
    L += (P != A && ecA[P] == cu[P]);
  }
  const bool posA = cu[A] > 0;
  auto allowed = [&](int B) { return (s.elig[B >> 5] >> (B & 31)) & 1u; };
  int bestg = -(1 << 20), bestB = k;
  for (int t = 0; t < nnp; ++t) {
    const int B = np[t];
    if (B == A || !allowed(B)) continue;
    const int cuB = cu[B];
    const int loseB = (cuB > 0 && ecA[B] == cuB) ? 1 : 0;
    const int new_ab = ecA[B] - cuB + cu[A];
    const int dab = (ecA[B] > 0 ? 1 : 0) - (new_ab > 0 ? 1 : 0);
    const unsigned* adjB = s.adjbits + (int64_t)B * W;
    int orv = 0;
    for (int t2 = 0; t2 < nnp && !orv; ++t2) {
      const int P = np[t2];
      orv = (P != B && !((adjB[P >> 5] >> (P & 31)) & 1u)) ? 1 : 0;
    }
    const int appear = orv - ((posA && !((adjB[A >> 5] >> (A & 31)) & 1u)) ? 1 : 0);
    const int g = L - loseB + dab - appear;
    if (g > bestg || (g == bestg && B < bestB)) {
      bestg = g;
      bestB = B;
    }
  }
  int f0 = -1, f1 = -1;
  for (int w = 0; w < W && f0 < 0; ++w) {
    unsigned base = s.elig[w];
    if ((A >> 5) == w) base &= ~(1u << (A & 31));
    for (int t = 0; t < nnp; ++t)
      if ((np[t] >> 5) == w) base &= ~(1u << (np[t] & 31));
    if (!base) continue;
    if (f1 < 0) f1 = w * 32 + __ffs(base) - 1;
    unsigned m0 = base;
    for (int t = 0; t < nnp && m0; ++t) m0 &= s.adjbits[(int64_t)np[t] * W + w];
    if (m0) f0 = w * 32 + __ffs(m0) - 1;
  }
  int fg = L, fB = f0;
  if (f0 < 0) {
    fg = L - 1;
    fB = f1;
  }
  if (fB >= 0 && (fg > bestg || (fg == bestg && fB < bestB))) {
    bestg = fg;
    bestB = fB;
  }
  if (bestB >= k) return 0ull;
  const unsigned long long flat = (unsigned long long)u * k + bestB;
  return ((unsigned long long)(bestg + (1ll << 20)) << 40) | ((1ull << 40) - 1 - flat);
}

__device__ bool fm_refine(PbrScratch& s, int n, int k, int* parts_io, unsigned long long* red64, long long* redll,
                          int* shflag) {
  // state: parts, conn (n x k), ec (k x k)
  for (int i = threadIdx.x; i < n; i += blockDim.x) s.parts[i] = parts_io[i];
  for (int64_t x = threadIdx.x; x < (int64_t)n * k; x += blockDim.x) s.conn[x] = 0;
  for (int64_t x = threadIdx.x; x < (int64_t)k * k; x += blockDim.x) s.ec[x] = 0;
  for (int p = threadIdx.x; p < k; p += blockDim.x) s.targets[p] = p < k - 1 ? kTile : n - kTile * (k - 1);
  __syncthreads();
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    for (int q = s.rowptr[u]; q < s.rowptr[u + 1]; ++q) {
      const int v = s.adj[q];
      s.conn[(int64_t)u * k + s.parts[v]] += 1;
      if (u < v) {  // each undirected edge once: ec[pa][pb] += 1, and ec[pb][pa] += 1 if pa != pb
        const int pa = s.parts[u], pb = s.parts[v];
        atomicAdd(&s.ec[(int64_t)pa * k + pb], 1);
        if (pa != pb) atomicAdd(&s.ec[(int64_t)pb * k + pa], 1);
      }
    }
  }
  __syncthreads();
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    int* l = s.npl + s.rowptr[u];
    int c = 0;
    for (int q = s.rowptr[u]; q < s.rowptr[u + 1]; ++q) {
      const int P = s.parts[s.adj[q]];
      bool seen = false;
      for (int t = 0; t < c; ++t) seen |= (l[t] == P);
      if (!seen) l[c++] = P;
    }
    s.npc[u] = c;
  }
  const int W = pbr_words(k);
  for (int64_t x = threadIdx.x; x < (int64_t)k * W; x += blockDim.x) {
    const int P = (int)(x / W), w = (int)(x - (int64_t)P * W);
    unsigned word = 0;
    for (int b = 0; b < 32; ++b) {
      const int Q = w * 32 + b;
      if (Q < k && Q != P && s.ec[(int64_t)P * k + Q] > 0) word |= 1u << b;
    }
    s.adjbits[x] = word;
  }
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    s.pmask[w] = 0;
    s.fmask[w] = 0;
  }
  if (threadIdx.x == 0) *s.flip = 0;
  __syncthreads();
  for (int pass = 0; pass < kMaxPasses; ++pass) {
    for (int p = threadIdx.x; p < k; p += blockDim.x) s.sizes[p] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      atomicAdd(&s.sizes[s.parts[i]], 1);
      s.locked[i] = 0;
      s.kvalid[i] = 0;
    }
    __syncthreads();
    long long badl = 0;
    for (int p = threadIdx.x; p < k; p += blockDim.x) badl += s.sizes[p] != s.targets[p];
    const bool start_bal = block_sum_i64(badl, redll) == 0;
    const long long start_obj = ec_objective(s, k, redll);
    bool have_best = start_bal;
    long long best = start_obj, cur = start_obj;
    int prefix = 0, hlen = 0, nlocked = 0;
    for (;;) {
      long long devbad = 0;
      for (int p = threadIdx.x; p < k; p += blockDim.x) devbad += s.sizes[p] != s.targets[p];
      const bool balanced = block_sum_i64(devbad, redll) == 0;
      // allowed destinations: every part when balanced, else the undersized ones
      for (int w = threadIdx.x; w < W; w += blockDim.x) {
        unsigned word = 0;
        for (int b = 0; b < 32; ++b) {
          const int B = w * 32 + b;
          if (B < k && (balanced || s.sizes[B] < s.targets[B])) word |= 1u << b;
        }
        s.elig[w] = word;
      }
      __syncthreads();
      unsigned long long key = 0;
      for (int attempt = 0; attempt < 2 && key == 0; ++attempt) {
        const bool ignore_locks = attempt == 1;
        if (balanced && ignore_locks) break;  // the lock-free fallback only applies when unbalanced
        for (int u = threadIdx.x; u < n; u += blockDim.x) {
          if (!ignore_locks && s.locked[u]) continue;
          unsigned long long kk;
          if (balanced) {
            // every destination allowed: the node's best move only changes when a move touched its
            // conn row, its part's ec row or an adjacency bit, so cached keys stay exact otherwise
            if (!s.kvalid[u]) {
              s.kcache[u] = fm_node_key(s, k, u);
              s.kvalid[u] = 1;
            }
            kk = s.kcache[u];
          } else {
            const int A = s.parts[u];
            if (!(s.sizes[A] > s.targets[A])) continue;
            kk = fm_node_key(s, k, u);
          }
          key = kk > key ? kk : key;
        }
        key = block_max_u64(key, red64);
      }
      if (key == 0) break;
      const unsigned long long flat = (1ull << 40) - 1 - (key & ((1ull << 40) - 1));
      const long long gain = (long long)(key >> 40) - (1ll << 20);
      const int u = (int)(flat / k), dst = (int)(flat % k);
      const int src = s.parts[u];
      __syncthreads();
      fm_move(s, k, u, dst);
      invalidate_marked(s, n, k);
      if (threadIdx.x == 0) {
        s.sizes[src] -= 1;
        s.sizes[dst] += 1;
        if (!s.locked[u]) *shflag = 1; else *shflag = 0;
        s.locked[u] = 1;
        s.hist[2 * hlen] = u;
        s.hist[2 * hlen + 1] = src;
        if (blockIdx.x == 0) {
          const int c = g_pbr_log[0];
          if (c < kLogMax) {
            g_pbr_log[1 + 4 * c] = u;
            g_pbr_log[2 + 4 * c] = dst;
            g_pbr_log[3 + 4 * c] = (int)gain;
            g_pbr_log[4 + 4 * c] = pass;
            g_pbr_log[0] = c + 1;
          }
        }
      }
      __syncthreads();
      nlocked += *shflag;
      cur -= gain;
      ++hlen;
      long long bad = 0;
      for (int p = threadIdx.x; p < k; p += blockDim.x) bad += s.sizes[p] != s.targets[p];
      const bool bal_now = block_sum_i64(bad, redll) == 0;
      if (bal_now && (!have_best || cur < best)) {
        have_best = true;
        best = cur;
        prefix = hlen;
      }
      if (nlocked == n) break;
    }
    for (int h = hlen - 1; h >= prefix; --h) {
      const int u = s.hist[2 * h], src = s.hist[2 * h + 1];
      const int dst = s.parts[u];
      fm_move(s, k, u, src);
      if (threadIdx.x == 0) {
        s.sizes[dst] -= 1;
        s.sizes[src] += 1;
      }
      __syncthreads();
    }
    const bool improved = (!start_bal && have_best) || (start_bal && have_best && best < start_obj);
    if (!improved) break;
  }
  long long bad = 0;
  for (int p = threadIdx.x; p < k; p += blockDim.x) bad += s.sizes[p] != s.targets[p];
  const bool ok = block_sum_i64(bad, redll) == 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) parts_io[i] = s.parts[i];
  __syncthreads();
  return ok;
}

// distinct unordered part pairs joined by an edge (partition_objective, reorder.py:112-119)
// and, with tiles = true, the number of non-empty t x t tiles (diagonal included).
__device__ long long pair_count(PbrScratch& s, int n, int k, const int* partof, bool tiles, long long* redll) {
  for (int64_t x = threadIdx.x; x < (int64_t)k * k; x += blockDim.x) s.ec[x] = 0;
  __syncthreads();
  for (int u = threadIdx.x; u < n; u += blockDim.x)
    for (int q = s.rowptr[u]; q < s.rowptr[u + 1]; ++q) {
      const int P = partof[u], Q = partof[s.adj[q]];
      if (tiles || P != Q) s.ec[(int64_t)P * k + Q] = 1;
    }
  __syncthreads();
  long long c = 0;
  for (int64_t x = threadIdx.x; x < (int64_t)k * k; x += blockDim.x) {
    const int P = (int)(x / k), Q = (int)(x - (int64_t)P * k);
    c += s.ec[x] && (tiles || P < Q);
  }
  return block_sum_i64(c, redll);
}

struct PbrGraph {
  int32_t n, S, k;
  int64_t node_off, scratch_off, tile_off, trow_off, nz_off;
  int64_t cand_stride;  // ints between the two candidates' scratch areas
};

// Adjacency from the octiles: rows in ascending column order == sorted unique neighbours
__device__ void build_adjacency(PbrScratch& s, const PbrGraph& g, const Octile* tiles, const int32_t* trow) {
  const int n = g.n;
  const Octile* t = tiles + g.tile_off;
  const int32_t* tr = trow + g.trow_off;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int I = i >> 3, r = i & 7;
    int c = 0;
    for (int q = tr[I]; q < tr[I + 1]; ++q) c += __popc((uint32_t)(t[q].bitmap >> (8 * r)) & 0xffu);
    s.tmp[i] = c;
    s.posmap[i] = -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < n; ++i) {
      s.rowptr[i] = acc;
      acc += s.tmp[i];
    }
    s.rowptr[n] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int I = i >> 3, r = i & 7;
    int pos = s.rowptr[i];
    for (int q = tr[I]; q < tr[I + 1]; ++q) {
      const Octile o = t[q];
      uint32_t byte = (uint32_t)(o.bitmap >> (8 * r)) & 0xffu;
      for (; byte; byte &= byte - 1) s.adj[pos++] = o.col * 8 + (__ffs(byte) - 1);
    }
  }
  __syncthreads();
}

// Phase 1: one CTA per (graph, candidate).  Candidate 0 is the natural order, candidate 1 the
// seeded SplitMix64 shuffle (reorder.py:385-393); each runs recursive bisection + K-way FM in its own
// scratch and leaves its partition in that scratch's cand[0..n).  The two candidates of a graph are
// independent, so they run on two SMs at once.
__global__ void __launch_bounds__(kPbrThreads) k_pbr_cand(const PbrGraph* __restrict__ gs, int G,
                                                         const Octile* tiles, const int32_t* trow, int* scratch,
                                                         uint64_t seed, int* status) {
  __shared__ unsigned long long red64[kPbrWarps];
  __shared__ long long redll[kPbrWarps];
  __shared__ int shw[kPbrWarps], shc, shi, shflag;
  for (int job = blockIdx.x; job < 2 * G; job += gridDim.x) {
    const int gi = job >> 1, c = job & 1;
    const PbrGraph g = gs[gi];
    const int n = g.n, k = g.k;
    if (k <= 1 || g.S == 0) continue;  // identity (k_pbr_finish)
    PbrScratch s = carve(scratch + g.scratch_off + c * g.cand_stride, n, g.S, k);
    build_adjacency(s, g, tiles, trow);
    for (int i = threadIdx.x; i < n; i += blockDim.x) s.order[i] = i;
    __syncthreads();
    if (c == 1 && threadIdx.x == 0) {
      SplitMix64 rng{seed};
      for (int i = n - 1; i > 0; --i) {
        const int j = (int)rng.randint((uint64_t)i + 1);
        const int x = s.order[i];
        s.order[i] = s.order[j];
        s.order[j] = x;
      }
    }
    __syncthreads();
    const long long c0 = clock64();
    recursive_parts(s, n, k, s.cand, red64, redll, shw, &shc, &shi);
    for (int i = threadIdx.x; i < n; i += blockDim.x) s.dbg[i] = s.cand[i];
    __syncthreads();
    const long long c1 = clock64();
    const bool ok = fm_refine(s, n, k, s.cand, red64, redll, &shflag);
    const long long c2 = clock64();
    if (threadIdx.x == 0) {
      atomicMax(&g_pbr_cycles[0], (unsigned long long)(c1 - c0));
      atomicMax(&g_pbr_cycles[1], (unsigned long long)(c2 - c1));
      if (!ok) atomicExch(status, 1);
    }
    __syncthreads();
  }
}

// Phase 2: one CTA per graph.  The candidate with the smaller Eq. 3 objective wins (natural on ties,
// reorder.py:394), nodes are ranked by (part, id) (permutation_from_partition, reorder.py:355-358), and
// the objective / octile-count fallbacks to identity apply (reorder.py:397-403).  Works in candidate
// 0's scratch (its adjacency is built).
__global__ void __launch_bounds__(kPbrThreads) k_pbr_finish(const PbrGraph* __restrict__ gs, int G, int* scratch,
                                                           int64_t* forward) {
  __shared__ long long redll[kPbrWarps];
  for (int gi = blockIdx.x; gi < G; gi += gridDim.x) {
    const PbrGraph g = gs[gi];
    const int n = g.n, k = g.k;
    int64_t* fwd = forward + g.node_off;
    if (k <= 1 || g.S == 0) {  // reorder.py:379-380
      for (int i = threadIdx.x; i < n; i += blockDim.x) fwd[i] = i;
      continue;
    }
    PbrScratch s = carve(scratch + g.scratch_off, n, g.S, k);
    const int* cand1 = carve(scratch + g.scratch_off + g.cand_stride, n, g.S, k).cand;
    const long long o0 = pair_count(s, n, k, s.cand, false, redll);
    const long long o1 = pair_count(s, n, k, cand1, false, redll);
    const int* best = (o0 <= o1) ? s.cand : cand1;  // min keeps the first on ties
    for (int p = threadIdx.x; p < k; p += blockDim.x) s.sizes[p] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&s.sizes[best[i]], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int p = 0; p < k; ++p) {
        const int c = s.sizes[p];
        s.sizes[p] = acc;
        acc += c;
      }
    }
    __syncthreads();
    // rank within a part by node id: count smaller ids in the same part
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int P = best[i];
      int r = 0;
      for (int j = 0; j < i; ++j) r += best[j] == P;
      s.tmp[i] = s.sizes[P] + r;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      s.side[i] = s.tmp[i] / kTile;  // parts of the permuted order
      s.locked[i] = i / kTile;       // identity parts
    }
    __syncthreads();
    const long long obj_perm = pair_count(s, n, k, s.side, false, redll);
    const long long obj_id = pair_count(s, n, k, s.locked, false, redll);
    bool use_perm = obj_perm <= obj_id;
    if (use_perm) {
      const long long tiles_perm = pair_count(s, n, k, s.side, true, redll);
      const long long tiles_id = pair_count(s, n, k, s.locked, true, redll);
      use_perm = tiles_perm <= tiles_id;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) fwd[i] = use_perm ? s.tmp[i] : i;
    __syncthreads();
  }
}

int pbr_device(int G, const std::vector<int64_t>& node_off, const std::vector<int64_t>& edge_off,
               const std::vector<int32_t>&, const std::vector<int32_t>&, uint64_t seed, const Octile* d_tiles,
               const std::vector<GraphDesc>& graphs, const int32_t* d_trow, int device, cudaStream_t stream,
               std::vector<int64_t>& forward, std::string& err) {
  (void)device;
  std::vector<PbrGraph> gs(G);
  int64_t off = 0;
  for (int g = 0; g < G; ++g) {
    const GraphDesc& d = graphs[g];
    PbrGraph p{};
    p.n = d.n;
    p.S = 2 * d.ne;
    p.k = (d.n + kTile - 1) / kTile;
    p.node_off = node_off[g];
    p.scratch_off = off;
    p.tile_off = d.tile_off;
    p.trow_off = d.trow_off;
    p.nz_off = d.nz_off;
    p.cand_stride = (pbr_scratch_ints(p.n, p.S, p.k) + 31) / 32 * 32;
    gs[g] = p;
    if (p.k > 1 && p.S > 0) off += 2 * p.cand_stride;
  }
  (void)edge_off;
  const int64_t nn = node_off[G];
  PbrGraph* d_gs = nullptr;
  int* d_scratch = nullptr;
  int64_t* d_fwd = nullptr;
  int* d_status = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_gs);
    cudaFree(d_scratch);
    cudaFree(d_fwd);
    cudaFree(d_status);
  };
  cudaError_t e = cudaMalloc(&d_gs, sizeof(PbrGraph) * G);
  if (e == cudaSuccess) e = cudaMalloc(&d_scratch, sizeof(int) * std::max<int64_t>(off, 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_fwd, sizeof(int64_t) * std::max<int64_t>(nn, 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_status, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_gs, gs.data(), sizeof(PbrGraph) * G, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_status, 0, sizeof(int), stream);
  if (e == cudaSuccess) {
    k_pbr_cand<<<2 * G, kPbrThreads, 0, stream>>>(d_gs, G, d_tiles, d_trow, d_scratch, seed, d_status);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
      k_pbr_finish<<<G, kPbrThreads, 0, stream>>>(d_gs, G, d_scratch, d_fwd);
      e = cudaGetLastError();
    }
  }
  int status = 0;
  forward.assign(nn, 0);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(forward.data(), d_fwd, sizeof(int64_t) * nn, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e == cudaSuccess && getenv("MGK_PBR_PROFILE")) {
    unsigned long long cyc[3] = {0, 0, 0};
    cudaMemcpyFromSymbol(cyc, g_pbr_cycles, sizeof(cyc));
    fprintf(stderr, "PBRPROF max cycles per candidate: bisection %llu, fm %llu\n", cyc[0], cyc[1]);
  }
  if (e == cudaSuccess && getenv("MGK_PBR_DEBUG")) {  // candidate partitions of every graph, for parity triage
    for (int g = 0; g < G; ++g) {
      if (gs[g].k <= 1 || gs[g].S == 0) continue;
      const int n = gs[g].n, S = gs[g].S, k = gs[g].k;
      std::vector<int> cand(2 * n), pre(2 * n);
      for (int c = 0; c < 2; ++c) {
        const int64_t base = gs[g].scratch_off + c * gs[g].cand_stride;
        const int64_t cand_off = base + (n + 1) + S + n;
        const int64_t dbg_off = base + pbr_scratch_ints(n, S, k) - 64 - 2 * (int64_t)n;
        cudaMemcpy(cand.data() + c * n, d_scratch + cand_off, sizeof(int) * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(pre.data() + c * n, d_scratch + dbg_off, sizeof(int) * n, cudaMemcpyDeviceToHost);
      }
      fprintf(stderr, "PBRDBG %d", g);
      for (int v : cand) fprintf(stderr, " %d", v);
      for (int v : pre) fprintf(stderr, " %d", v);
      fprintf(stderr, "\n");
    }
    std::vector<int> lg(1 + 4 * kLogMax);
    cudaMemcpyFromSymbol(lg.data(), g_pbr_log, sizeof(int) * lg.size());
    fprintf(stderr, "PBRLOG");
    for (int i = 0; i < 1 + 4 * std::min(lg[0], kLogMax); ++i) fprintf(stderr, " %d", lg[i]);
    fprintf(stderr, "\n");
  }
  cleanup();
  if (e != cudaSuccess) {
    err = std::string("pbr: ") + cudaGetErrorString(e);
    return MGK_E_CUDA;
  }
  if (status) {
    err = "FM refinement failed to restore balance";
    return MGK_E_INVALID;
  }
  return MGK_OK;
}

}  // namespace mgk

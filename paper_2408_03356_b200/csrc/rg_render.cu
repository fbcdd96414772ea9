// rg_render.cu -- slab-by-slab volume ray casting of the Gaussians through the
// BVH, forward and backward:
//
//   PAPER.md Alg. 2: per ray, bbox clip, then slabs of B samples
//   of length dt*B; per slab the set of Gaussians whose support overlaps the
//   slab (Alg. 1 any-hit collection, capped at K = n_max with the
//   K smallest (t_entry, index) kept -- DESIGN.md L7), sorted by entry depth;
//   UpdateRay = evaluate sigma and the density-weighted colour at the B
//   samples (Eq. 10-16) and composite front to back (Eq. 4); early
//   termination at slab granularity when T <= T_eps.
//
// B200 design: ONE WARP PER RAY.  The ray keeps a sorted
// ACTIVE LIST (shared memory, capacity kA) of its upcoming/overlapping
// Gaussians with their per-pair data (exact interval, weight-exponent
// polynomial, colour), refilled by a warp-cooperative k-nearest-by-t_entry
// traversal of the 32-wide BVH ("next k keys after a cursor"): one node visit
// = 32 lanes testing the node's 32 child boxes, leaf children tested exactly
// by their lane, the k-buffer held one key per lane (rank/ballot merge),
// internal children pushed nearest-last on a shared stack.  Empty slabs are
// skipped exactly (jump to the slab holding the next t_entry).  Integration
// maps lanes to (entry-subset x sample) and reduces with shuffles;
// compositing is a segmented scan over the slab's samples with the optical
// depth accumulated (Kahan) so T does not drift over thousands of samples.
// Backward replays the same march, walks each sample group front to back with
// suffix = P - prefix (L16), accumulates per-pair moments in shared memory
// and scatters each pair's 16 + app_stride gradient floats as one coalesced
// burst of float4 atomics (one per lane) into a Morton-ordered buffer;
// k_finalize converts (mu, M) -> (mu, q, s) and un-permutes.
#include "rg_internal.cuh"
#include <cuda_fp16.h>

#include <type_traits>

namespace rg {

namespace {

#ifndef RG_EVAL_UNROLL
#define RG_EVAL_UNROLL 4         // forward window evaluation loop (sweep: 1 +2%, 2 +0.8%)
#endif
#ifndef RG_EVAL_BRANCHFREE
#define RG_EVAL_BRANCHFREE 1     // window evaluation predicated, not branched (medians of 9:
#endif                           // forward 7.243 -> 6.797 ms; profiles/r2/ab_eval_branchfree.log)
#ifndef RG_GRAD_BRANCHFREE
#define RG_GRAD_BRANCHFREE 1     // backward member loop predicated (medians of 9: backward
#endif                           // 5.558 -> 5.025 ms; profiles/r2/ab_grad_branchfree.log)
#ifndef RG_PREFETCH_APP
#define RG_PREFETCH_APP 0        // restart query: prefetch candidates' appearance records (A/B)
#endif
#ifndef RG_STORE_WINDOWS
#define RG_STORE_WINDOWS 1       // forward stores the 4-slab windows' sums for the backward
#endif
#ifndef RG_TWO_UNCOND
#define RG_TWO_UNCOND 0          // restart query: the second node's loads without a branch
#endif
#ifndef RG_GRAD_FIXED
#define RG_GRAD_FIXED 0          // backward member loop over the whole part (A/B knob)
#endif
#ifndef RG_RANGE_BRANCHFREE
#define RG_RANGE_BRANCHFREE 1    // per-slab-path evaluation (eval_range) predicated in the
#endif                           // backward (medians of 9: backward 5.18 -> 5.02 ms; the
                                 // forward is faster branched, 6.93 vs 6.79 ms)
#ifndef RG_P2_MIN
#define RG_P2_MIN 4              // backward window pass: smallest member group (4 or 8 lanes)
#endif
#ifndef RG_SH_ONE_PAIR
#define RG_SH_ONE_PAIR 0         // backward SH scatter: 0 = two pairs per iteration (half-warps)
#endif
#ifndef RG_SG_HALF_ITEMS
#define RG_SG_HALF_ITEMS 0       // backward SG scatter items: 0 = (pair, lobe), 1 = (pair, lobe, half)
#endif
#ifndef RG_MEMBER_UNROLL
#define RG_MEMBER_UNROLL 2       // backward member loop
#endif
#ifndef RG_MIN_BLOCKS
#define RG_MIN_BLOCKS 4                // resident blocks per SM the register budget targets (bwd)
#endif
#ifndef RG_MIN_BLOCKS_FWD
// forward, 64-slot list (no WarpAcc: smem allows more blocks): 5 blocks -> 96 registers,
// 20 warps/SM; medians of 9 (profiles/r2/ab_fwd_blocks.log): C1 forward 6.76 -> 6.36 ms
// with 5, 6.76 with 6 (80 registers, 144 B of spills); the 128-slot list keeps 4 (C3
// forward 230 -> 251 ms with 5)
#define RG_MIN_BLOCKS_FWD 5
#endif
constexpr int kEvalUnroll = RG_EVAL_UNROLL;
constexpr int kMemberUnroll = RG_MEMBER_UNROLL;
constexpr int kWarps = 4;              // rays (warps) per block
static_assert(kWarps == 4, "camera mode: a block is a 2x2 pixel tile, or one pixel's 4 subsamples");
constexpr int kBlock = 32 * kWarps;
constexpr int kA = 64;                 // persistent active-list capacity
constexpr int kTrans = kA;             // transient chunk slots (slab sets > kA)
constexpr int kRet = kA + 32;          // retired (expired, not yet scattered) slots, backward
constexpr int kSlots = kA + 64;
static_assert(kA == 64, "expire/n_in handle two 32-slot chunks");
#ifndef RG_STK_FWD
#define RG_STK_FWD 256
#endif
// traversal stack entries (wide nodes; max depth seen (tools/probe_stack.sh): C1 60,
// C3 135; an overflow drops subtrees and is counted in rg_stats.stack_overflows,
// asserted 0 by the tests): the forward takes 256 (320: +0.8% forward, 512: +1%
// more, through the smaller L1 carve-out); the
// backward traverses only for rays whose fetch log overflowed and must stay within
// its 48 KB block budget
constexpr int kStkFwd = RG_STK_FWD;
constexpr int kStkBwd = 192;   // C4 re-traversals need it (168 overflowed: stress gradients off)
constexpr unsigned kFull = 0xffffffffu;

struct Counters {
  uint32_t slabs, pairs, evals, samples, overflows, fetches, nodes, stackov, restarts;
};

struct RenderArgs {
  SceneView S;
  rg_config c;
  int cam_mode;
  rg_camera cam;
  int rw, rh, tiles_x;
  const float* ro;
  const float* rd;
  int n_rays;
  float* rgb;
  float* T;
  int32_t* replay;
  int32_t* log;            // per-ray fetch records [n_rays, kLogWords] (forward writes)
  float4* arena;           // pair slots (3 float4 each)
  unsigned long long* arena_ctr;
  long long arena_cap;     // slots
  int pair_fix;            // pair slots owned by each ray (arena [0, n_rays * pair_fix))
  float4* samp;            // per-window sample sums (sigma, sigma c_r, c_g, c_b), 32 per window
  unsigned long long* samp_ctr;
  long long samp_cap;      // float4 units
  rg_stats* stats;
  int dbg_rays, dbg_cap;
  int32_t* dbg_counts;
  int32_t* dbg_rec;
  // backward
  const float* rgb_in;
  const int32_t* replay_in;
  const float* d_rgb;
  float* gbuf;
  int gstride;
};

// per-slot entry (AoS, three float4 so a lane reads a slot with LDS.128):
//   e0 = {t_entry, t_exit, t_mid, c0}   e1 = {c1, c2, r, g}   e2 = {b, pos, idx, -}
// per-ray state of the persistent traversal (stream_next, below)
struct Stream {
  int nf, qn, ch, cn;                 // frontier size, queued leaves, candidate head / count
  unsigned long long lim, c0;         // completeness bound, restart cursor
  bool valid;
};

#ifndef RG_STK64
#define RG_STK64 0   // restart-query stack entries as one 8-B word (medians of 9: forward
                     // 6.231 -> 6.304 ms; kept as an A/B knob)
#endif
template <int STK, int NCAP, int CCAP, int KA = kA, int SLOTS = kSlots>
struct WarpMemT {
  static constexpr int kStack = STK;
  static constexpr bool k64 = RG_STK64 != 0 && STK <= 256;   // the 520-list keeps 6-B entries
  static constexpr int kNCap = NCAP;
  static constexpr int kCCap = CCAP;
  static constexpr int kList = KA;     // active-list capacity
  static constexpr int kNSlots = SLOTS;
  static constexpr int kTr = KA;       // first transient slot (restart-query scratch)
  float4 e0[SLOTS], e1[SLOTS], e2[SLOTS];
  union {
    struct {             // restart query (fetch)
      uint2 st2[k64 ? STK : 1];   // {wide node id, 16-bit entry key}: one 8-B access
      uint32_t stk[k64 ? 1 : STK];   // or: stacked wide node ids
      uint16_t stn[k64 ? 1 : STK];   // their boxes' entry distances as 16-bit order keys
                                     // (fp16 rounded down): pop-time selection and pruning
    } r;
    struct {             // persistent per-ray traversal (stream_next); clobbered by fetch
      uint32_t nk[NCAP];   // node frontier: fkey of a lower bound on every t_entry below
      uint32_t nid[NCAP];  //   the node, and the wide node id (unsorted)
      unsigned long long ck[CCAP];   // exact-tested candidates, sorted by (t_entry key, index)
      uint32_t cp[CCAP];   //   and their Morton positions
      uint32_t lqk[NCAP > 1 ? 96 : 1];   // box-entry lower bounds of the queued leaves (fkey)
    } s;
  } u;
  // queued Gaussians awaiting the exact test (fetch): kept in the transient slots'
  // e2 words, dead during a query; < 32 left over + the leaf ranges of kLqGroup
  // lanes at a time
  static constexpr int kLq = (SLOTS - KA) * 4;
  static constexpr int kLqGroup = 31 + 32 * kLeafRange <= kLq ? 32 : 31 + 16 * kLeafRange <= kLq ? 16 : 8;
  static_assert(31 + kLqGroup * kLeafRange <= kLq, "leaf queue");
#if RG_STREAM
  uint32_t lq[96];     // stream_next's leaf queue
#endif
  Stream sst;          // stream_next state between refills (registers only inside the call)
  // fetch-log bookkeeping of the ray (warp-uniform, rarely touched): kept here, not in
  // registers, to relieve the register pressure of the march loops
  struct { int lp, nwin, wcur, fix; int ok, wl; } ls;
  alignas(16) float Y[16];   // Y(d) of the ray (zero past the degree), read as float4 by the scatter
};
// Persistent per-ray traversal (stream_next) for the forward refills: built, measured
// and kept as a compile-time option (RG_STREAM=1), OFF by default: it cut C1 node visits
// by 35% but was slower (C1 forward 7.1 -> 9.5-10.2 ms, C3 334 -> 554 ms: its frontier
// bookkeeping costs more per visit and C3 rays hit ~1000 distinct wide nodes anyway, so
// the restarts it removes were not the cost)
#ifndef RG_STREAM
#define RG_STREAM 0
#endif
#ifndef RG_NCAP
#define RG_NCAP 192
#endif
#ifndef RG_CCAP
#define RG_CCAP 96
#endif
#ifndef RG_STREAM_FROM
#define RG_STREAM_FROM 0       // forward refills served by restart queries before the stream
#endif
constexpr bool kStream = RG_STREAM != 0;
static_assert(!kStream || kLeafRange == 1, "stream_next queues single leaves (RG_LEAF_RANGE=1)");
constexpr int kNCap = kStream ? RG_NCAP : 1;   // forward node-frontier capacity (stream_next)
constexpr int kCCap = kStream ? RG_CCAP : 32;  // forward candidate capacity (stream_next)
static_assert(kCCap % 32 == 0 && kCCap <= 128, "candidate merge reads CCAP/32 entries per lane");
using WMFwd = WarpMemT<kStkFwd, kNCap, kCCap>;
using WMBwd = WarpMemT<kStkBwd, 1, 1>;     // the backward refills by restart queries only
// forward "large list" variant (rg_config.list_capacity > 64): an active list that holds
// every member of a slab up to K = 519 (C4 stress: per-slab sets of ~1000, K = 512), so
// truncated slabs take the K held smallest keys instead of streaming the rest of every
// slab with restart queries (C4: 7750 -> ~100 queries per ray); two 4-warp blocks per SM
constexpr int kABig = 520;
using WMBig = WarpMemT<320, 1, 32, kABig, kABig + 32>;
// a medium list (rg_config.list_capacity 65..128): per-slab sets of up to 128 without
// streaming, four blocks per SM (C3: slab sets above 64 Gaussians are common)
constexpr int kAMid = 128;
using WMMid = WarpMemT<kStkFwd, 1, 32, kAMid, kAMid + 64>;
using WMBwdMid = WarpMemT<kStkBwd, 1, 1, kAMid, kAMid + 64>;
template <int SLOTS, bool HASC = true>
struct WarpAccT {
  float4 a[SLOTS];     // Sw, Sw1, Sw2, dc_r
  float2 b[SLOTS];     // dc_g, dc_b
  float c[HASC ? SLOTS : 1];   // sum w dL/dw (dL/dsigma~ of non-Gaussian bases; the
                               // Gaussian's is a.x, so its kernels do not allocate it)
  float4 s0[32];
  float s1[32];        // per-sample backward values of the current group / window:
                          // {tk, dls, dc0, dc1}, {dc2, gc, inv, live}
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
  const unsigned lo = __shfl_sync(kFull, (unsigned)v, src);
  const unsigned hi = __shfl_sync(kFull, (unsigned)(v >> 32), src);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long shfl64x(unsigned long long v, int mask) {
  const unsigned lo = __shfl_xor_sync(kFull, (unsigned)v, mask);
  const unsigned hi = __shfl_xor_sync(kFull, (unsigned)(v >> 32), mask);
  return ((unsigned long long)hi << 32) | lo;
}

// conservative ray/AABB overlap (sign-selected slabs: empty boxes never hit)
__device__ __forceinline__ void box_t(float lx, float ly, float lz, float hx, float hy, float hz,
                                      const float3& inv, const float3& oinv, float& tn, float& tf) {
  const float ax = fmaf(lx, inv.x, -oinv.x), bx = fmaf(hx, inv.x, -oinv.x);
  const float ay = fmaf(ly, inv.y, -oinv.y), by = fmaf(hy, inv.y, -oinv.y);
  const float az = fmaf(lz, inv.z, -oinv.z), bz = fmaf(hz, inv.z, -oinv.z);
  const float nx = inv.x >= 0.f ? ax : bx, fx = inv.x >= 0.f ? bx : ax;
  const float ny = inv.y >= 0.f ? ay : by, fy = inv.y >= 0.f ? by : ay;
  const float nz = inv.z >= 0.f ? az : bz, fz = inv.z >= 0.f ? bz : az;
  tn = fmaxf(fmaxf(nx, ny), nz);
  tf = fminf(fminf(fx, fy), fz);
}

struct Ray {
  float3 o, d, inv, oinv;
};


// entry distance <-> order-preserving 16-bit key (fp16 rounded toward -inf:
// a decoded key never exceeds the distance, so pruning on it is conservative)
__device__ __forceinline__ uint16_t stn_enc(float t) {
  const unsigned b = __half_as_ushort(__float2half_rd(t));
  return (uint16_t)((b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u));
}
__device__ __forceinline__ float stn_dec(unsigned k) {
  const unsigned b = (k & 0x8000u) ? (k & 0x7FFFu) : (~k & 0xFFFFu);
  return __half2float(__ushort_as_half((unsigned short)b));
}

template <class WM>
__device__ __forceinline__ void stk_put(WM& M, int i, uint32_t nid, unsigned k16) {
  if constexpr (WM::k64) M.u.r.st2[i] = make_uint2(nid, k16);
  else { M.u.r.stk[i] = nid; M.u.r.stn[i] = (uint16_t)k16; }
}
template <class WM>
__device__ __forceinline__ void stk_get(const WM& M, int i, uint32_t& nid, unsigned& k16) {
  if constexpr (WM::k64) {
    const uint2 e = M.u.r.st2[i];
    nid = e.x; k16 = e.y;
  } else {
    nid = M.u.r.stk[i]; k16 = M.u.r.stn[i];
  }
}

// Warp-cooperative k-nearest query on the 32-wide BVH: the kmax (<= 32)
// smallest keys (t_entry bits, index) > cursor among Gaussians whose exact
// support interval satisfies t_exit >= seg_lo and t_entry <= seg_hi.
// Result: lane l < return value holds the l-th smallest key and its position.
// KEYCMP: pop-time pruning in the 16-bit key domain (forward: medians of 9, 6.355 ->
// 6.231 ms); the backward keeps the float compare (its register budget: 4.83 vs 4.91 ms)
template <class WM, bool KEYCMP = true>
__device__ int fetch(const SceneView& S, WM& M, const Ray& R, float seg_lo, float seg_hi,
                     unsigned long long cursor, int kmax, unsigned long long& key, uint32_t& pos,
                     Counters& cnt) {
  const unsigned lane = lane_id();
  const unsigned lt_mask = (1u << lane) - 1u;
  if (lane == 0) cnt.fetches++;
  // candidate sort scratch aliases the transient slots, dead during every fetch
  unsigned long long* const kscr = reinterpret_cast<unsigned long long*>(&M.e0[WM::kTr]);
  uint32_t* const pscr = reinterpret_cast<uint32_t*>(&M.e1[WM::kTr]);
  uint32_t* const lq = reinterpret_cast<uint32_t*>(&M.e2[WM::kTr]);
  key = ~0ull;
  pos = 0;
  int nk = 0;
  float te_lim = INFINITY;
  // pop-time pruning in the 16-bit key domain: stn_dec(k) > te_lim + slack  <=>
  // k > stn_enc(te_lim + slack) (stn_enc rounds down to the largest fp16 <= its
  // argument, stn_dec is strictly monotone; the bound is never -0: slack > 0)
  unsigned klim = KEYCMP ? stn_enc(INFINITY) : 0u;
  unsigned long long kth = ~0ull;
  const float slack = 1e-5f * (fabsf(seg_lo) + fabsf(seg_hi)) + 1e-6f;
  const float lo_s = seg_lo - slack, hi_s = seg_hi + slack;
  int sp = 1, qn = 0;
  if (lane == 0) stk_put(M, 0, 0u, stn_enc(-INFINITY));
  __syncwarp();
  // Exact leaf tests are batched: box-passing leaves are queued in shared
  // memory and tested 32 at a time (all lanes busy), then the candidates are
  // bitonic-sorted and bitonic-merged into the k-buffer.
  // ---- fq exact test
  auto flush = [&](int off, int n) {   // exact tests of lq[off, off + n), n <= 32
    __syncwarp();
    const uint32_t cp = (int)lane < n ? lq[off + lane] : 0u;
    bool cand = false;
    unsigned long long ck = ~0ull;
    if ((int)lane < n) {
      const float4* gp = S.geom + 4 * (size_t)cp;
      const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2), g3 = __ldg(gp + 3);
      PairGeom pg;
      if (isect_exact(g0, g1, g2, g3, R.o, R.d, pg) && pg.tx >= seg_lo && pg.te <= seg_hi) {
        ck = ((unsigned long long)fkey(pg.te) << 32) | (uint32_t)__float_as_int(g3.z);
        cand = ck > cursor && ck < kth;
        if (!cand) ck = ~0ull;
#if RG_PREFETCH_APP
        if (cand) {   // its appearance record is read by the set-up if it survives the query
          const char* ap = reinterpret_cast<const char*>(S.app + (size_t)cp * S.app_stride);
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            if (RG_PREFETCH_APP == 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(ap + 128 * l));
            else asm volatile("prefetch.global.L2 [%0];" ::"l"(ap + 128 * l));
          }
        }
#endif
      }
    }
    const unsigned cmask = __ballot_sync(kFull, cand);
    if (!cmask) return;
    uint32_t cpos;
    const int ncand = __popc(cmask);
    // ---- fq rank sort
    // sort the candidates by rank (O(#candidates)): place, then read back in order
    // (a 32-bit-key variant for distinct t_entry keys, MATCH + vote first, measured
    // no faster: forward 7.247 -> 7.281 ms, medians of 9)
    {
      int crank = 0;
      unsigned mm = cmask;
      while (mm) {
        const int b = __ffs(mm) - 1;
        mm &= mm - 1;
        const unsigned long long kb = shfl64(ck, b);
        crank += (cand && kb < ck) ? 1 : 0;
      }
      RG_CHECK(!cand || crank < 32);
      if (cand) { kscr[crank] = ck; pscr[crank] = cp; }
      __syncwarp();
      ck = (int)lane < ncand ? kscr[lane] : ~0ull;
      cpos = pscr[lane];
      __syncwarp();
    }
    // ---- fq merge
    // the 32 smallest of (k-buffer, candidates) form a bitonic sequence: merge
    {
      const unsigned long long rk = shfl64(ck, 31 - (int)lane);
      const uint32_t rp = __shfl_sync(kFull, cpos, 31 - (int)lane);
      if (rk < key) { key = rk; pos = rp; }
    }
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
      const unsigned long long ok = shfl64x(key, j);
      const uint32_t op = __shfl_xor_sync(kFull, pos, j);
      if ((((int)lane & j) == 0) ? (ok < key) : (ok > key)) { key = ok; pos = op; }
    }
    if ((int)lane >= kmax) { key = ~0ull; pos = 0u; }
    nk = __popc(__ballot_sync(kFull, key != ~0ull));
    if (nk == kmax) {
      kth = shfl64(key, kmax - 1);
      te_lim = fkey_inv((uint32_t)(kth >> 32));
      if (KEYCMP) klim = stn_enc(te_lim + slack);
    }
  };
  // ---- fq drain
  // exact tests of the full 32-entry groups; the < 32 left over move to the front
  auto drain = [&]() {
    if (qn < 32) return;
    int off = 0;
    do { flush(off, 32); off += 32; } while (qn - off >= 32);
    const int rem = qn - off;
    const uint32_t mv = (int)lane < rem ? lq[off + lane] : 0u;
    __syncwarp();
    if ((int)lane < rem) lq[lane] = mv;
    qn = rem;
  };
  // queue the Gaussians of one node's hit leaf ranges (lane order), kLqGroup lanes
  // at a time
  auto enqueue = [&](bool lf, int child) {
    const int f0 = leaf_range_first(child);
#pragma unroll
    for (int g = 0; g < 32; g += WM::kLqGroup) {
      if (g) drain();
      const bool in = lf && (int)lane >= g && (int)lane < g + WM::kLqGroup;
      const int c = in ? leaf_range_count(child) : 0;
      int inc = c;                                    // inclusive warp scan of the counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, inc, o);
        if ((int)lane >= o) inc += v;
      }
      const int tot = __shfl_sync(kFull, inc, 31);
      RG_CHECK(qn + tot <= WM::kLq);
      const int w = qn + inc - c;
#pragma unroll
      for (int r = 0; r < kLeafRange; ++r)
        if (r < c) lq[w + r] = (uint32_t)(f0 + r);
      qn += tot;
      __syncwarp();
    }
  };
  // Best-first-ish DFS: each iteration pops the two nodes with the smallest entry
  // distances among the top 32 stack entries and visits both (their 14 child-box
  // loads per lane are in flight together); when even the nearest lies beyond the
  // k-th key, all 32 are dropped.  Pushes are unordered (the pop selects).
  while (sp > 0) {
    // ---- fq pop
    int nodeA, nodeB = -1;
    {
      const int nwin = min(sp, 32);
      unsigned k16 = 0xFFFFu, nid = 0;
      if ((int)lane < nwin) stk_get(M, sp - 1 - (int)lane, nid, k16);
      // (key, lane) packed: one reduction yields the minimum and its lane (ties
      // to the lowest lane; a key reduction + ballot + ffs was 2.2% slower)
      const unsigned kl = (k16 << 5) | lane;
      const unsigned klmin = __reduce_min_sync(kFull, kl);
      const unsigned kmin = klmin >> 5;
      if (KEYCMP ? kmin > klim : stn_dec(kmin) > te_lim + slack) {
        sp -= nwin;
        continue;
      }
      const int srcA = (int)(klmin & 31u);
      nodeA = (int)__shfl_sync(kFull, nid, srcA);
      int srcB = -1;
#ifndef RG_ONE_NODE
      const unsigned k16b = (int)lane == srcA ? 0xFFFFu : k16;
      const unsigned klmin2 = __reduce_min_sync(kFull, (k16b << 5) | lane);
      const unsigned kmin2 = klmin2 >> 5;
      if (KEYCMP ? kmin2 <= klim                      // (empty lanes: 0xFFFF > klim)
                 : kmin2 != 0xFFFFu && stn_dec(kmin2) <= te_lim + slack) {
        srcB = (int)(klmin2 & 31u);
        nodeB = (int)__shfl_sync(kFull, nid, srcB);
      }
#endif
      // remove the popped entries: the surviving top entries (lanes 0, 1) fill the
      // holes the popped ones leave further down
      if (srcB < 0) {
        if (lane == 0 && srcA != 0) stk_put(M, sp - 1 - srcA, nid, k16);
        sp -= 1;
      } else {
        const bool m0 = srcA != 0 && srcB != 0, m1 = srcA != 1 && srcB != 1;
        const int h1 = srcA >= 2 ? srcA : srcB, h2 = srcA >= 2 ? srcB : srcA;   // holes (>= 2 first)
        int hole = -1;
        if (lane == 0 && m0) hole = h1;
        if (lane == 1 && m1) hole = m0 ? h2 : h1;
        if (hole >= 2) stk_put(M, sp - 1 - hole, nid, k16);
        sp -= 2;
      }
      __syncwarp();
    }
    if (lane == 0) cnt.nodes += nodeB >= 0 ? 2 : 1;
    const bool two = nodeB >= 0;
    // ---- fq node loads
    const WideNode& WA = S.wide[nodeA];
    const WideNode& WB = S.wide[two ? nodeB : nodeA];
    const int childA = __ldg(&WA.child[lane]);
    const float alx = __ldg(&WA.lox[lane]), aly = __ldg(&WA.loy[lane]), alz = __ldg(&WA.loz[lane]);
    const float ahx = __ldg(&WA.hix[lane]), ahy = __ldg(&WA.hiy[lane]), ahz = __ldg(&WA.hiz[lane]);
#if RG_TWO_UNCOND
    // node B loaded unconditionally (node A again when there is no second node: L1
    // hits), its children masked: no branch around the loads
    int childB = __ldg(&WB.child[lane]);
    const float blx = __ldg(&WB.lox[lane]), bly = __ldg(&WB.loy[lane]), blz = __ldg(&WB.loz[lane]);
    const float bhx = __ldg(&WB.hix[lane]), bhy = __ldg(&WB.hiy[lane]), bhz = __ldg(&WB.hiz[lane]);
    if (!two) childB = kWideEmpty;
#else
    int childB = kWideEmpty;
    float blx = 0.f, bly = 0.f, blz = 0.f, bhx = 0.f, bhy = 0.f, bhz = 0.f;
    if (two) {
      childB = __ldg(&WB.child[lane]);
      blx = __ldg(&WB.lox[lane]); bly = __ldg(&WB.loy[lane]); blz = __ldg(&WB.loz[lane]);
      bhx = __ldg(&WB.hix[lane]); bhy = __ldg(&WB.hiy[lane]); bhz = __ldg(&WB.hiz[lane]);
    }
#endif
    // ---- fq box test
    float tnA, tfA, tnB, tfB;
    box_t(alx, aly, alz, ahx, ahy, ahz, R.inv, R.oinv, tnA, tfA);
    box_t(blx, bly, blz, bhx, bhy, bhz, R.inv, R.oinv, tnB, tfB);
    const bool hitA = childA != kWideEmpty && tnA <= tfA && tfA >= lo_s && tnA <= hi_s &&
                      tnA <= te_lim + slack;
    const bool hitB = childB != kWideEmpty && tnB <= tfB && tfB >= lo_s && tnB <= hi_s &&
                      tnB <= te_lim + slack;
    // ---- fq leaf queue
    // queue the Gaussians of box-passing leaf ranges (A's, then B's)
    {
      const bool lfA = hitA && childA < 0, lfB = hitB && childB < 0;
      const unsigned lmA = __ballot_sync(kFull, lfA);
      const unsigned lmB = __ballot_sync(kFull, lfB);
      if (lmA | lmB) {
        __syncwarp();
        if (kLeafRange == 1) {
          RG_CHECK(qn + __popc(lmA) + __popc(lmB) <= WM::kLq);
          if (lfA) lq[qn + __popc(lmA & lt_mask)] = (uint32_t)leaf_range_first(childA);
          if (lfB) lq[qn + __popc(lmA) + __popc(lmB & lt_mask)] = (uint32_t)leaf_range_first(childB);
          qn += __popc(lmA) + __popc(lmB);
        } else {
          enqueue(lfA, childA);
          if (lmB) {
            drain();                                  // < 32 left before B's ranges
            enqueue(lfB, childB);
          }
        }
      }
    }
    // ---- fq push
    // internal children, any order (the pop selects)
    const unsigned imA = __ballot_sync(kFull, hitA && childA >= 0);
    const unsigned imB = __ballot_sync(kFull, hitB && childB >= 0);
    if (imA | imB) {
      const int npA = __popc(imA), np = npA + __popc(imB);
      __syncwarp();
      if (sp + np <= WM::kStack) {
        if (hitA && childA >= 0) {
          const int r = sp + __popc(imA & lt_mask);
          stk_put(M, r, (uint32_t)childA, stn_enc(tnA));
        }
        if (hitB && childB >= 0) {
          const int r = sp + npA + __popc(imB & lt_mask);
          stk_put(M, r, (uint32_t)childB, stn_enc(tnB));
        }
        sp += np;
#ifdef RG_STACK_PROBE
        if (lane == 0 && (uint32_t)sp > cnt.stackov) cnt.stackov = sp;   // max depth, not overflows
#endif
      } else if (lane == 0) {
        cnt.stackov++;
      }
      __syncwarp();
    }
    drain();
  }
  for (int off = 0; off < qn; off += 32) flush(off, min(qn - off, 32));
  return nk;
}

// ---------------------------------------------------------------------------
// Persistent per-ray traversal of the forward refills: an incremental
// best-first search (Hjaltason & Samet's incremental nearest neighbour) that
// emits the ray's Gaussians in exact key order (t_entry bits, index) and
// expands every wide node at most once per ray -- the restart query `fetch`
// re-descends from the root for every refill (C3 rays refill 12.5 times and
// revisit the nodes of every Gaussian still alive).  State kept in shared
// memory between the refills of a ray:
//   NF  unexpanded wide nodes, each with a lower bound on every t_entry below it
//       (the box entry minus the box-test slack);
//   LQ  box-passing leaves queued for the batched exact test, with the same bound;
//   CF  exact-tested candidates, sorted by key.
// A candidate is emitted only when its key lies below every NF / LQ bound, so
// the emission order is the exact key order and the per-slab sets are those of
// the restart query.  A frontier or candidate overflow drops the largest new
// entries and lowers `lim`: the state is complete only below lim, and reaching
// lim restarts from the root with the last emitted key as the cursor (bounded
// memory, still exact).  `fetch` (restart queries of the overflow paths)
// clobbers this state: the caller then clears `valid`.


template <class WM>
__device__ __forceinline__ void stream_restart(WM& M, Stream& st, unsigned long long cursor) {
  if (lane_id() == 0) { M.u.s.nk[0] = 0u; M.u.s.nid[0] = 0u; }
  st.nf = 1; st.qn = 0; st.ch = 0; st.cn = 0;
  st.lim = ~0ull; st.c0 = cursor; st.valid = true;
  __syncwarp();
}

// exact test of the first n queued leaves, merge of the hits into CF
template <class WM>
__device__ __forceinline__ void stream_flush(const SceneView& S, WM& M, Stream& st, const Ray& R,
                                             float tlo, float t1, int n) {
  constexpr int CCAP = WM::kCCap;
  const unsigned lane = lane_id();
  unsigned long long* const kscr = reinterpret_cast<unsigned long long*>(&M.e0[WM::kTr]);
  uint32_t* const pscr = reinterpret_cast<uint32_t*>(&M.e1[WM::kTr]);
  uint32_t* const lq = reinterpret_cast<uint32_t*>(&M.e2[WM::kTr]);
  __syncwarp();
  const uint32_t cp = (int)lane < n ? M.lq[lane] : 0u;
  bool cand = false;
  unsigned long long ck = ~0ull;
  if ((int)lane < n) {
    const float4* gp = S.geom + 4 * (size_t)cp;
    const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2), g3 = __ldg(gp + 3);
    PairGeom pg;
    if (isect_exact(g0, g1, g2, g3, R.o, R.d, pg) && pg.tx >= tlo && pg.te <= t1) {
      ck = ((unsigned long long)fkey(pg.te) << 32) | (uint32_t)__float_as_int(g3.z);
      cand = ck > st.c0 && ck < st.lim;
      if (!cand) ck = ~0ull;
    }
  }
  // drop the consumed queue entries
  {
    const int rem = st.qn - n;   // < 64 left over
    const uint32_t mv = (int)lane < rem ? M.lq[n + lane] : 0u;
    const uint32_t mv2 = (int)lane + 32 < rem ? M.lq[n + 32 + lane] : 0u;
    const uint32_t mk = (int)lane < rem ? M.u.s.lqk[n + lane] : 0u;
    const uint32_t mk2 = (int)lane + 32 < rem ? M.u.s.lqk[n + 32 + lane] : 0u;
    __syncwarp();
    if ((int)lane < rem) { M.lq[lane] = mv; M.u.s.lqk[lane] = mk; }
    if ((int)lane + 32 < rem) { M.lq[32 + lane] = mv2; M.u.s.lqk[32 + lane] = mk2; }
    st.qn = rem;
  }
  const unsigned cmask = __ballot_sync(kFull, cand);
  if (!cmask) { __syncwarp(); return; }
  const int nc = __popc(cmask);
  // rank sort of the new candidates into kscr/pscr [0, nc)
  {
    int crank = 0;
    unsigned mm = cmask;
    while (mm) {
      const int b = __ffs(mm) - 1;
      mm &= mm - 1;
      const unsigned long long kb = shfl64(ck, b);
      crank += (cand && kb < ck) ? 1 : 0;
    }
    if (cand) { kscr[crank] = ck; pscr[crank] = cp; }
  }
  __syncwarp();
  // merge with the sorted CF [ch, ch + cn): destination = own rank + rank in the other list
  unsigned long long ok[CCAP / 32];
  uint32_t op[CCAP / 32];
  int od[CCAP / 32];
#pragma unroll
  for (int t = 0; t < CCAP / 32; ++t) {
    const int i = (int)lane + 32 * t;
    ok[t] = ~0ull; op[t] = 0u; od[t] = CCAP;
    if (i < st.cn) {
      ok[t] = M.u.s.ck[st.ch + i];
      op[t] = M.u.s.cp[st.ch + i];
      int lo = 0, len = nc;               // new keys < ok[t]
      while (len > 0) {
        const int half = len >> 1;
        if (kscr[lo + half] < ok[t]) { lo += half + 1; len -= half + 1; } else { len = half; }
      }
      od[t] = i + lo;
    }
  }
  unsigned long long nk_ = ~0ull;
  uint32_t np_ = 0u;
  int nd = CCAP;
  if ((int)lane < nc) {
    nk_ = kscr[lane];
    np_ = pscr[lane];
    int lo = 0, len = st.cn;              // old keys < nk_
    while (len > 0) {
      const int half = len >> 1;
      if (M.u.s.ck[st.ch + lo + half] < nk_) { lo += half + 1; len -= half + 1; } else { len = half; }
    }
    nd = (int)lane + lo;
  }
  __syncwarp();
  unsigned long long dropped = ~0ull;
#pragma unroll
  for (int t = 0; t < CCAP / 32; ++t) {
    if (od[t] < CCAP) { M.u.s.ck[od[t]] = ok[t]; M.u.s.cp[od[t]] = op[t]; }
    else if (ok[t] < dropped) dropped = ok[t];
  }
  if (nd < CCAP) { M.u.s.ck[nd] = nk_; M.u.s.cp[nd] = np_; }
  else if (nk_ < dropped) dropped = nk_;
  const int tot = st.cn + nc;
  st.ch = 0;
  st.cn = min(tot, CCAP);
  if (tot > CCAP) {            // complete only below the smallest dropped key
    unsigned long long v = dropped;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = shfl64x(v, off);
      v = o < v ? o : v;
    }
    if (v < st.lim) st.lim = v;
  }
  __syncwarp();
}

// next `want` (<= 32) keys of the ray after `cursor` (lane l < return value
// holds the l-th key and its position); fewer than `want` = exhausted
template <class WM>
__device__ int stream_next(const SceneView& S, WM& M, const Ray& R, float tlo, float t1,
                           unsigned long long cursor, int want, unsigned long long& key,
                           uint32_t& pos, Counters& cnt) {
  constexpr int NCAP = WM::kNCap;
  const unsigned lane = lane_id();
  const unsigned lt_mask = (1u << lane) - 1u;
  if (lane == 0) cnt.fetches++;
  key = ~0ull;
  pos = 0;
  int got = 0;
  Stream st = M.sst;
  if (!st.valid) stream_restart(M, st, cursor);
  const float slack = 1e-5f * (fabsf(tlo) + fabsf(t1)) + 1e-6f;
  const float hi_s = t1 + slack;
  float lo_b = tlo;
  if (st.c0 != 0ull) lo_b = fmaxf(lo_b, fkey_inv((uint32_t)(st.c0 >> 32)));
  lo_b -= slack;
  while (true) {
    // lower bounds: the two smallest node keys (with slots) and the smallest queued leaf
    unsigned a1 = ~0u, a2 = ~0u;
    int s1 = 0, s2 = 0;
    for (int j = (int)lane; j < st.nf; j += 32) {
      const unsigned k = M.u.s.nk[j];
      if (k < a1) { a2 = a1; s2 = s1; a1 = k; s1 = j; }
      else if (k < a2) { a2 = k; s2 = j; }
    }
    unsigned qmin = ~0u;
    for (int j = (int)lane; j < st.qn; j += 32) qmin = min(qmin, M.u.s.lqk[j]);
    const unsigned mN = __reduce_min_sync(kFull, a1);
    const unsigned mQ = __reduce_min_sync(kFull, qmin);
    const unsigned m = min(mN, mQ);
    const bool open_any = st.nf > 0 || st.qn > 0;
    unsigned long long bound = open_any ? ((unsigned long long)m << 32) : ~0ull;
    if (st.lim < bound) bound = st.lim;
    // emit the candidates below every bound (CF is sorted: a prefix)
    {
      const bool can = (int)lane < min(st.cn, 32) && M.u.s.ck[st.ch + (int)lane] < bound;
      const int e = min(__popc(__ballot_sync(kFull, can)), want - got);
      if ((int)lane >= got && (int)lane < got + e) {
        key = M.u.s.ck[st.ch + (int)lane - got];
        pos = M.u.s.cp[st.ch + (int)lane - got];
      }
      st.ch += e;
      st.cn -= e;
      got += e;
      if (got == want) break;
    }
    // everything still open lies at or beyond lim: drop it
    if (open_any && st.lim != ~0ull && ((unsigned long long)m << 32) >= st.lim) {
      st.nf = 0;
      st.qn = 0;
      continue;
    }
    if (!open_any) {
      if (st.lim == ~0ull) break;                       // exhausted
      // complete only below lim, and every key below lim has been emitted: restart
      // from the root after max(last emitted key, lim - 1)
      const unsigned long long last = got > 0 ? shfl64(key, got - 1) : cursor;
      const unsigned long long c0n = last > st.lim - 1 ? last : st.lim - 1;
      if (c0n <= st.c0) {
        // no progress since the last restart (a frontier that cannot hold the ray's
        // nearby nodes): finish this call with a restart query (always terminates)
        unsigned long long fk;
        uint32_t fp;
        const int g2 = fetch(S, M, R, tlo, t1, last, want - got, fk, fp, cnt);
        const int src = (int)lane - got;
        const unsigned long long mk = shfl64(fk, src & 31);
        const uint32_t mp = __shfl_sync(kFull, fp, src & 31);
        if (src >= 0 && src < g2) { key = mk; pos = mp; }
        got += g2;
        st.valid = false;                               // fetch reused the traversal memory
        break;
      }
      stream_restart(M, st, c0n);
      lo_b = fmaxf(tlo, fkey_inv((uint32_t)(c0n >> 32))) - slack;
      if (lane == 0) cnt.restarts++;
      continue;
    }
    // exact-test queued leaves when they bound the emission or fill a batch
    if (st.qn > 0 && (mQ <= mN || st.qn >= 32)) {
      stream_flush(S, M, st, R, tlo, t1, min(st.qn, 32));
      continue;
    }
    // expand the nearest node and, if there is one, the second nearest
    const int srcA = __ffs(__ballot_sync(kFull, a1 == mN)) - 1;
    const int slotA = __shfl_sync(kFull, s1, srcA);
    const unsigned c2 = (int)lane == srcA ? a2 : a1;
    const int sl2 = (int)lane == srcA ? s2 : s1;
    const unsigned mN2 = __reduce_min_sync(kFull, c2);
    int slotB = -1;
    if (mN2 != ~0u && ((unsigned long long)mN2 << 32) < st.lim) {
      const int srcB = __ffs(__ballot_sync(kFull, c2 == mN2)) - 1;
      slotB = __shfl_sync(kFull, sl2, srcB);
    }
    const int nodeA = (int)M.u.s.nid[slotA];
    const int nodeB = slotB >= 0 ? (int)M.u.s.nid[slotB] : -1;
    __syncwarp();
    if (lane == 0) {        // remove the popped slots (the larger first): the last entry fills
      int h1 = slotA, h2 = slotB;
      if (h2 > h1) { const int t = h1; h1 = h2; h2 = t; }
      int nf = st.nf;
      if (h1 != nf - 1) { M.u.s.nk[h1] = M.u.s.nk[nf - 1]; M.u.s.nid[h1] = M.u.s.nid[nf - 1]; }
      --nf;
      if (h2 >= 0) {
        if (h2 != nf - 1) { M.u.s.nk[h2] = M.u.s.nk[nf - 1]; M.u.s.nid[h2] = M.u.s.nid[nf - 1]; }
        --nf;
      }
    }
    st.nf -= nodeB >= 0 ? 2 : 1;
    __syncwarp();
    if (lane == 0) cnt.nodes += nodeB >= 0 ? 2 : 1;
    const bool two = nodeB >= 0;
    const WideNode& WA = S.wide[nodeA];
    const WideNode& WB = S.wide[two ? nodeB : nodeA];
    const int childA = __ldg(&WA.child[lane]);
    const float alx = __ldg(&WA.lox[lane]), aly = __ldg(&WA.loy[lane]), alz = __ldg(&WA.loz[lane]);
    const float ahx = __ldg(&WA.hix[lane]), ahy = __ldg(&WA.hiy[lane]), ahz = __ldg(&WA.hiz[lane]);
    int childB = kWideEmpty;
    float blx = 0.f, bly = 0.f, blz = 0.f, bhx = 0.f, bhy = 0.f, bhz = 0.f;
    if (two) {
      childB = __ldg(&WB.child[lane]);
      blx = __ldg(&WB.lox[lane]); bly = __ldg(&WB.loy[lane]); blz = __ldg(&WB.loz[lane]);
      bhx = __ldg(&WB.hix[lane]); bhy = __ldg(&WB.hiy[lane]); bhz = __ldg(&WB.hiz[lane]);
    }
    float tnA, tfA, tnB, tfB;
    box_t(alx, aly, alz, ahx, ahy, ahz, R.inv, R.oinv, tnA, tfA);
    box_t(blx, bly, blz, bhx, bhy, bhz, R.inv, R.oinv, tnB, tfB);
    const uint32_t kA_ = fkey(tnA - slack), kB_ = fkey(tnB - slack);
    const unsigned lim_hi = (unsigned)(st.lim >> 32);
    const bool hitA = childA != kWideEmpty && tnA <= tfA && tfA >= lo_b && tnA <= hi_s && kA_ <= lim_hi;
    const bool hitB = childB != kWideEmpty && tnB <= tfB && tfB >= lo_b && tnB <= hi_s && kB_ <= lim_hi;
    {   // queue box-passing leaves (A's, then B's)
      const unsigned lmA = __ballot_sync(kFull, hitA && childA < 0);
      const unsigned lmB = __ballot_sync(kFull, hitB && childB < 0);
      if (lmA | lmB) {
        if (hitA && childA < 0) {
          const int r = st.qn + __popc(lmA & lt_mask);
          M.lq[r] = (uint32_t)(~childA); M.u.s.lqk[r] = kA_;
        }
        if (hitB && childB < 0) {
          const int r = st.qn + __popc(lmA) + __popc(lmB & lt_mask);
          M.lq[r] = (uint32_t)(~childB); M.u.s.lqk[r] = kB_;
        }
        st.qn += __popc(lmA) + __popc(lmB);
      }
    }
    {   // internal children join the frontier; those beyond its capacity lower lim
      const unsigned imA = __ballot_sync(kFull, hitA && childA >= 0);
      const unsigned imB = __ballot_sync(kFull, hitB && childB >= 0);
      if (imA | imB) {
        const int npA = __popc(imA), np = npA + __popc(imB);
        unsigned dk = ~0u;
        if (hitA && childA >= 0) {
          const int r = st.nf + __popc(imA & lt_mask);
          if (r < NCAP) { M.u.s.nk[r] = kA_; M.u.s.nid[r] = (uint32_t)childA; } else dk = kA_;
        }
        if (hitB && childB >= 0) {
          const int r = st.nf + npA + __popc(imB & lt_mask);
          if (r < NCAP) { M.u.s.nk[r] = kB_; M.u.s.nid[r] = (uint32_t)childB; } else dk = min(dk, kB_);
        }
        if (st.nf + np > NCAP) {
          const unsigned dmin = __reduce_min_sync(kFull, dk);
          const unsigned long long l2 = (unsigned long long)dmin << 32;
          if (l2 < st.lim) st.lim = l2;
        }
        st.nf = min(st.nf + np, NCAP);
      }
    }
    __syncwarp();
  }
  __syncwarp();
  if (lane == 0) M.sst = st;
  __syncwarp();
  return got;
}

// c_l(d) = sum_m c~_m Y_m(d) + sum_j k_j e^{lambda_j (d.p_j - 1)} (Eq. 14-15):
// Y(d) is per-ray in shared memory (zero past the degree, so the fixed 16-
// coefficient SH region of the record needs no predicate); SG lobes at 48+7j.
// VEC: 16-B loads (forward: -5% time); scalar loads in the backward, where the
// extra registers of the vector form cost more (+3%) than they save
template <bool VEC>
__device__ __forceinline__ float3 pair_color(const SceneView& S, const float* Y, int pos,
                                             const float3& d) {
  if (!VEC) {
  const float* ap = S.app + (size_t)pos * S.app_stride;
  float r = 0.f, g = 0.f, b = 0.f;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    r = fmaf(Y[m], __ldg(ap + 3 * m), r);
    g = fmaf(Y[m], __ldg(ap + 3 * m + 1), g);
    b = fmaf(Y[m], __ldg(ap + 3 * m + 2), b);
  }
  for (int j = 0; j < S.lobes; ++j) {
    const float* q = ap + kShFloats + 7 * j;
    const float dp = d.x * __ldg(q + 4) + d.y * __ldg(q + 5) + d.z * __ldg(q + 6);
    const float e = ex2_approx(__ldg(q + 3) * (dp - 1.0f) * kLog2e);
    r = fmaf(__ldg(q), e, r);
    g = fmaf(__ldg(q + 1), e, g);
    b = fmaf(__ldg(q + 2), e, b);
  }
  return make_float3(r, g, b);
  }
  // 16-B loads: the record is 16-B aligned, SH [m][3] in floats 0..47, lobe j in
  // floats 48+7j..54+7j (2 or 3 float4s, neighbours re-read from L1)
  const float4* a4 = reinterpret_cast<const float4*>(S.app + (size_t)pos * S.app_stride);
  float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < kShFloats / 4; ++i) {
    const float4 v = __ldg(a4 + i);
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int f = 4 * i + k;
      acc[f % 3] = fmaf(Y[f / 3], vv[k], acc[f % 3]);
    }
  }
  const int L = S.lobes;
#pragma unroll
  for (int j = 0; j < kMaxLobes; ++j) {
    if (j >= L) break;
    const int f0 = kShFloats + 7 * j;           // compile-time after unrolling
    const int i0 = f0 / 4, i1 = (f0 + 6) / 4;   // float4s covering the lobe (2 or 3)
    float w[12];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i0 + i <= i1) {
        const float4 v = __ldg(a4 + i0 + i);
        w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
      }
    }
    const float* p = w + (f0 - 4 * i0);
    const float dp = d.x * p[4] + d.y * p[5] + d.z * p[6];
    const float e = ex2_approx(p[3] * (dp - 1.0f) * kLog2e);
    acc[0] = fmaf(p[0], e, acc[0]);
    acc[1] = fmaf(p[1], e, acc[1]);
    acc[2] = fmaf(p[2], e, acc[2]);
  }
  return make_float3(acc[0], acc[1], acc[2]);
}

// Per-(ray, Gaussian) set-up into slot `sl`: exact interval and the exponent
// polynomial of w(tau) = sigma~ exp(-|u + tau d_l|^2 / 2) = 2^(c0 + tau (c1 + c2 tau)),
// tau = t - t_mid, u = M x' from the compensated offset x' (value path).
// inlined: a call would save/restore the caller's ~128 live registers (measured
// slower: fwd 10.97 -> 10.31 ms, bwd 11.92 -> 11.69 ms on C1 when inlined)
#ifdef RG_NOINLINE_SETUP
#define RG_SETUP_ATTR __noinline__
#else
#define RG_SETUP_ATTR __forceinline__
#endif
#ifdef RG_NOINLINE_SCATTER
#define RG_SCATTER_ATTR __noinline__
#else
#define RG_SCATTER_ATTR __forceinline__
#endif
// ---- basis functions (supplementary P:456-515).  Gaussian slots hold
// log2 w(tau) = c0 + tau (c1 + c2 tau); other bases hold q(tau) = |M x(tau)|^2 =
// qm + tau (2 b1 + A tau) (e0.w, e1.x, e1.y) and sigma~ (e2.w).
template <int BASIS>
__device__ __forceinline__ float basis_w(float tau, const float4& a, const float4& q, float sig,
                                         float& qq) {
  const float p = fmaf(tau, fmaf(q.y, tau, q.x), a.w);
  qq = p;
  if (BASIS == 0) return ex2_approx(p);
  const float pp = fmaxf(p, 0.f);
  if (BASIS == 1) return pp < 1.f ? sig * ex2_approx((1.f - 1.f / (1.f - pp)) * kLog2e) : 0.f;
  if (BASIS == 2) {
    const float r = sqrtf(pp), u = 1.f - r;
    return r <= 1.f ? sig * ((u * u) * (u * u)) * fmaf(4.f, r, 1.f) : 0.f;
  }
  if (BASIS == 3) return sig * rsqrtf(1.f + pp);
  if (BASIS == 4) return sig / (1.f + pp);
  return sig * ex2_approx(-sqrtf(pp) * kLog2e);                    // C0-Matern
}
// psi = -2 sigma~ dphi/dq (dw/dy = -psi y); the Gaussian's psi is w
template <int BASIS>
__device__ __forceinline__ float basis_psi(float w, float qq, float sig) {
  if (BASIS == 0) return w;
  const float pp = fmaxf(qq, 0.f);
  if (BASIS == 1) { const float u = 1.f - pp; return pp < 1.f ? 2.f * w / (u * u) : 0.f; }
  if (BASIS == 2) {
    const float r = sqrtf(pp), u = 1.f - r;
    return r <= 1.f ? 20.f * sig * (u * u * u) : 0.f;
  }
  if (BASIS == 3) { const float ph = w / sig; return w * ph * ph; }     // sigma~ (1+q)^-3/2
  if (BASIS == 4) return 2.f * w * (w / sig);                           // 2 sigma~ (1+q)^-2
  const float r = sqrtf(pp);
  return r > 0.f ? w / r : 0.f;                                         // kink at r = 0
}

template <bool VEC, int BASIS, class WM>
__device__ RG_SETUP_ATTR void setup_pair(const SceneView& S, WM& M, int sl, const Ray& R,
                                        uint32_t pos) {
  RG_CHECK(sl >= 0 && sl < WM::kNSlots && (int)pos < S.n);
  const float4* gp = S.geom + 4 * (size_t)pos;
  const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2), g3 = __ldg(gp + 3);
  PairGeom pg;
  isect_exact(g0, g1, g2, g3, R.o, R.d, pg);
  const float x0 = offset_at(R.o.x, g0.x, pg.tm, R.d.x);
  const float x1 = offset_at(R.o.y, g0.y, pg.tm, R.d.y);
  const float x2 = offset_at(R.o.z, g0.z, pg.tm, R.d.z);
  const float u0 = g1.x * x0 + g1.y * x1 + g1.z * x2;
  const float u1 = g1.w * x0 + g2.x * x1 + g2.y * x2;
  const float u2 = g2.z * x0 + g2.w * x1 + g3.x * x2;
  const float qm = u0 * u0 + u1 * u1 + u2 * u2;
  const float b1 = u0 * pg.dl0 + u1 * pg.dl1 + u2 * pg.dl2;
  const float3 col = pair_color<VEC>(S, M.Y, (int)pos, R.d);
  if (BASIS == 0) {
    M.e0[sl] = make_float4(pg.te, pg.tx, pg.tm, lg2_approx(g0.w) - 0.5f * kLog2e * qm);
    M.e1[sl] = make_float4(-kLog2e * b1, -0.5f * kLog2e * pg.A, col.x, col.y);
    M.e2[sl] = make_float4(col.z, __int_as_float((int)pos), g3.z, 0.f);
  } else {
    M.e0[sl] = make_float4(pg.te, pg.tx, pg.tm, qm);
    M.e1[sl] = make_float4(2.f * b1, pg.A, col.x, col.y);
    M.e2[sl] = make_float4(col.z, __int_as_float((int)pos), g3.z, g0.w);
  }
}

// 1 - exp(-x) without cancellation for small x (both forms, then a select: no branch)
__device__ __forceinline__ float alpha_of(float x, float e) {
  const float ser = x * (1.f - 0.5f * x * (1.f - (1.f / 3.f) * x * (1.f - 0.25f * x)));
  return x < 0.0625f ? ser : 1.0f - e;
}

// lane -> (entry subset esub, sample j) for one group of GW samples
template <int GW>
struct Lanes {
  static constexpr int ER = 32 / GW;
  int j, esub;
};

// sigma and sigma*c at this lane's sample from slots [e0, e1)
template <int GW, int BASIS, bool PRED, class WM>
__device__ __forceinline__ void eval_range(const WM& M, int e0, int e1, const Lanes<GW>& L,
                                           float tk, bool val, float& s, float& r, float& g,
                                           float& b, uint32_t& evals) {
  float2 rg2 = make_float2(r, g);
#if RG_RANGE_BRANCHFREE
  if (BASIS == 0 && PRED) {
#pragma unroll 2
    for (int e = e0 + L.esub; e < e1; e += Lanes<GW>::ER) {
      const float4 a = M.e0[e];
      const float4 q = M.e1[e];
      const float cb = M.e2[e].x;
      const float tau = tk - a.z;
      const float wv = ex2_approx(fmaf(tau, fmaf(q.y, tau, q.x), a.w));
      const bool in = val && a.x <= tk && tk <= a.y;
      const float w = in ? wv : 0.f;
      s += w;
      rg2 = __ffma2_rn(make_float2(w, w), make_float2(q.z, q.w), rg2);
      b = fmaf(w, cb, b);
      evals += in ? 1u : 0u;
    }
    r = rg2.x;
    g = rg2.y;
    return;
  }
#endif
#pragma unroll 2
  for (int e = e0 + L.esub; e < e1; e += Lanes<GW>::ER) {
    const float4 a = M.e0[e];
    if (val && a.x <= tk && tk <= a.y) {
      const float4 q = M.e1[e];
      const float cb = M.e2[e].x;
      const float sge = BASIS != 0 ? M.e2[e].w : 0.f;   // sigma~ (non-Gaussian slots)
      const float tau = tk - a.z;
      float qq;
      const float w = basis_w<BASIS>(tau, a, q, sge, qq);
      s += w;
      rg2 = __ffma2_rn(make_float2(w, w), make_float2(q.z, q.w), rg2);
      b = fmaf(w, cb, b);
      ++evals;
    }
  }
  r = rg2.x;
  g = rg2.y;
}

struct SampleGrad {   // per-sample backward quantities (lanes of sample j)
  float dls, dc0, dc1, dc2, gc, inv;
};

// accumulate the per-pair moments of slots [e0, e1) over this group's samples:
// lane = slot, loop over the GW samples whose backward values the composite
// step left in A.s0/A.s1 (broadcast reads), moments kept in registers.
template <int GW, int BASIS, class WM, class AC>
__device__ __forceinline__ void grad_range(const WM& M, AC& A, int e0, int e1) {
  __syncwarp();
  for (int base = e0; base < e1; base += 32) {
    const int e = base + (int)lane_id();
    if (e < e1) {
      const float4 a = M.e0[e];
      const float4 q = M.e1[e];
      const float cb = M.e2[e].x;
      const float sge = BASIS != 0 ? M.e2[e].w : 0.f;   // sigma~ (non-Gaussian slots)
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f;
#pragma unroll
      for (int j = 0; j < GW; ++j) {
        const float4 s0 = A.s0[j];
        const float tk = s0.x;
        if (a.x <= tk && tk <= a.y) {
          const float b2 = A.s1[j];
          const float tau = tk - a.z;
          float qq;
          const float w = basis_w<BASIS>(tau, a, q, sge, qq);
          const float dldw = fmaf(s0.z, q.z, fmaf(s0.w, q.w, fmaf(b2, cb, s0.y)));
          const float wd = basis_psi<BASIS>(w, qq, sge) * dldw;
          a0 += wd;
          a1 = fmaf(wd, tau, a1);
          a2 = fmaf(wd * tau, tau, a2);
          a3 = fmaf(w, s0.z, a3);
          a4 = fmaf(w, s0.w, a4);
          a5 = fmaf(w, b2, a5);
          if (BASIS != 0) a6 = fmaf(w, dldw, a6);
        }
      }
      float4 v = A.a[e];
      float2 w = A.b[e];
      v.x += a0; v.y += a1; v.z += a2; v.w += a3;
      w.x += a4; w.y += a5;
      A.a[e] = v;
      A.b[e] = w;
      if (BASIS != 0) A.c[e] += a6;
    }
  }
  __syncwarp();
}

// Gradient scatter of the slots in `mask` (relative to `base`), warp-cooperative:
//  geometry: each lane owning a slot computes its 13 values, 4 float4 atomics;
//  appearance: per slot, lane c writes chunk 4 + c (one coalesced burst).
//  With x = x' + tau d, u = M x', d_l = M d and Sw = sum w dL/dw, Sw1 = sum w dL/dw tau,
//  Sw2 = sum w dL/dw tau^2:  dL/dmu = M^T (Sw u + Sw1 d_l),
//  dL/dM = -(Sw u x'^T + Sw1 (u d^T + d_l x'^T) + Sw2 d_l d^T),  dL/dsigma~ = Sw / sigma~.
template <int BASIS, class WM, class AC>
__device__ RG_SCATTER_ATTR void scatter_batch(const SceneView& S, const WM& M, const AC& A,
                                           int base, unsigned mask, const Ray& R,
                                           float* gbuf, int gstride) {
  const unsigned lane = lane_id();
  const int qsh = sh_pad(S.deg) / 4;   // float4 chunks per SH channel
  // drop slots with all-zero moments (never contributed)
  {
    bool nz = false;
    if (mask & (1u << lane)) {
      const float4 v = A.a[base + lane];
      const float2 w = A.b[base + lane];
      nz = v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f || w.x != 0.f || w.y != 0.f ||
           (BASIS != 0 && A.c[BASIS != 0 ? base + lane : 0] != 0.f);
    }
    mask = __ballot_sync(kFull, nz);
  }
  if (!mask) return;
  if (mask & (1u << lane)) {
    const int e = base + (int)lane;
    const float4 acc = A.a[e];
    const float Sw = acc.x, Sw1 = acc.y, Sw2 = acc.z;
    const float4 x0 = M.e0[e];
    const int pos = __float_as_int(M.e2[e].y);
    const float4 g0 = __ldg(S.geom + 4 * (size_t)pos);
    const float tm = x0.z;
    const float xp[3] = {offset_at(R.o.x, g0.x, tm, R.d.x), offset_at(R.o.y, g0.y, tm, R.d.y),
                         offset_at(R.o.z, g0.z, tm, R.d.z)};
    const float dv[3] = {R.d.x, R.d.y, R.d.z};
    // M-free sufficient statistics (linear in the pair's moments, summed over rays):
    //   v = Sw x' + Sw1 d,  S = Sw x'x'^T + Sw1 (x'd^T + d x'^T) + Sw2 d d^T (symmetric);
    // k_finalize forms dL/dmu = M^T M v and dL/dM = -M S once per Gaussian
    const float v0 = fmaf(Sw, xp[0], Sw1 * dv[0]);
    const float v1 = fmaf(Sw, xp[1], Sw1 * dv[1]);
    const float v2 = fmaf(Sw, xp[2], Sw1 * dv[2]);
    const float h0 = fmaf(Sw2, dv[0], Sw1 * xp[0]);   // Sw1 x' + Sw2 d
    const float h1 = fmaf(Sw2, dv[1], Sw1 * xp[1]);
    const float h2 = fmaf(Sw2, dv[2], Sw1 * xp[2]);
    // S_ab = x'_a (Sw x'_b + Sw1 d_b) + d_a (Sw1 x'_b + Sw2 d_b) = x'_a v_b + d_a h_b
    const float s00 = fmaf(xp[0], v0, dv[0] * h0);
    const float s01 = fmaf(xp[0], v1, dv[0] * h1);
    const float s02 = fmaf(xp[0], v2, dv[0] * h2);
    const float s11 = fmaf(xp[1], v1, dv[1] * h1);
    const float s12 = fmaf(xp[1], v2, dv[1] * h2);
    const float s22 = fmaf(xp[2], v2, dv[2] * h2);
    RG_CHECK(pos >= 0 && pos < S.n);
    float4* row = reinterpret_cast<float4*>(gbuf + (size_t)pos * gstride);
    atomicAdd(row + 0, make_float4(v0, v1, v2, (BASIS == 0 ? Sw : A.c[BASIS != 0 ? e : 0]) / g0.w));
    atomicAdd(row + 1, make_float4(s00, s01, s02, s11));
    atomicAdd(row + 2, make_float4(s12, s22, 0.f, 0.f));
  }
#if RG_SG_HALF_ITEMS
  // SG lobes: lane = (pair, lobe, half) item (RG_SG_HALF_ITEMS=1): every half
  // re-evaluates its lobe, twice the items of the per-lobe form
  if (S.lobes > 0) {
    const int per = 2 * S.lobes;
    const float inv_per = 1.0f / (float)per;
    const int nitems = (32 - __clz(mask)) * per;
    const int c0 = 3 * qsh;                           // first SG chunk of the row
    for (int it = (int)lane; it - (int)lane < nitems; it += 32) {
      int b = (int)((float)it * inv_per);             // it / per (small ints), corrected
      if (b * per > it) --b;
      if ((b + 1) * per <= it) ++b;
      const int c = it - b * per;
      if (it < nitems && ((mask >> b) & 1u)) {
        const int e = base + b;
        const float4 acc = A.a[e];
        const float2 acb = A.b[e];
        const float d0 = acc.w, d1 = acb.x, d2 = acb.y;
        const int pos = __float_as_int(M.e2[e].y);
        const float* q = S.app + (size_t)pos * S.app_stride + kShFloats + 7 * (c >> 1);
        const float lam = __ldg(q + 3);
        const float dpm = R.d.x * __ldg(q + 4) + R.d.y * __ldg(q + 5) + R.d.z * __ldg(q + 6) - 1.0f;
        const float ej = ex2_approx(lam * dpm * kLog2e);
        const float kd = (d0 * __ldg(q) + d1 * __ldg(q + 1) + d2 * __ldg(q + 2)) * ej;
        float4 v;
        if ((c & 1) == 0) {
          v = make_float4(d0 * ej, d1 * ej, d2 * ej, kd * dpm);
        } else {
          const float kdl = kd * lam;
          v = make_float4(kdl * R.d.x, kdl * R.d.y, kdl * R.d.z, 0.f);
        }
        atomicAdd(reinterpret_cast<float4*>(gbuf + (size_t)pos * gstride) + 4 + c0 + c, v);
      }
    }
  }
#else
  // SG lobes: lane = (pair, lobe) item, so several pairs' record loads are in flight
  // per instruction (the per-pair loop below waits on one pair at a time); the item
  // evaluates its lobe once and issues both halves (k, lambda | p) of its gradient
  if (S.lobes > 0) {
    const int per = S.lobes;
    const float inv_per = 1.0f / (float)per;
    const int nitems = (32 - __clz(mask)) * per;
    const int c0 = 3 * qsh;                           // first SG chunk of the row
    for (int it = (int)lane; it - (int)lane < nitems; it += 32) {
      int b = (int)((float)it * inv_per);             // it / per (small ints), corrected
      if (b * per > it) --b;
      if ((b + 1) * per <= it) ++b;
      const int c = it - b * per;
      if (it < nitems && ((mask >> b) & 1u)) {
        const int e = base + b;
        const float4 acc = A.a[e];
        const float2 acb = A.b[e];
        const float d0 = acc.w, d1 = acb.x, d2 = acb.y;
        const int pos = __float_as_int(M.e2[e].y);
        const float* q = S.app + (size_t)pos * S.app_stride + kShFloats + 7 * c;
        const float lam = __ldg(q + 3);
        const float dpm = R.d.x * __ldg(q + 4) + R.d.y * __ldg(q + 5) + R.d.z * __ldg(q + 6) - 1.0f;
        const float ej = ex2_approx(lam * dpm * kLog2e);
        const float kd = (d0 * __ldg(q) + d1 * __ldg(q + 1) + d2 * __ldg(q + 2)) * ej;
        const float kdl = kd * lam;
        float4* dst = reinterpret_cast<float4*>(gbuf + (size_t)pos * gstride) + 4 + c0 + 2 * c;
        atomicAdd(dst, make_float4(d0 * ej, d1 * ej, d2 * ej, kd * dpm));
        atomicAdd(dst + 1, make_float4(kdl * R.d.x, kdl * R.d.y, kdl * R.d.z, 0.f));
      }
    }
  }
#endif
  // SH: one coalesced burst per pair, lane = (channel, 4 coefficients):
  // dL/dc~_m = dc[ch] Y_m(d), Y(d) from shared memory (zero past the degree).
  // A burst is 3 * pad4(nc) / 4 <= 12 lanes, so each half-warp takes a pair
  // (RG_SH_ONE_PAIR=1: one pair per iteration, 20 lanes idle)
#if RG_SH_ONE_PAIR
  const int ch = (int)lane < 3 * qsh ? (int)lane / qsh : -1;
  float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ch >= 0) y = *reinterpret_cast<const float4*>(&M.Y[4 * ((int)lane - ch * qsh)]);
  while (mask) {
    const int b = __ffs(mask) - 1;
    mask &= mask - 1;
    const int e = base + b;
    const int pos = __float_as_int(M.e2[e].y);
    if (ch >= 0) {
      const float dsel = ch == 0 ? A.a[e].w : (ch == 1 ? A.b[e].x : A.b[e].y);
      atomicAdd(reinterpret_cast<float4*>(gbuf + (size_t)pos * gstride) + 4 + lane,
                make_float4(dsel * y.x, dsel * y.y, dsel * y.z, dsel * y.w));
    }
  }
#else
  const int l16 = (int)lane & 15;
  const bool upper = lane >= 16u;
  const int ch = l16 < 3 * qsh ? l16 / qsh : -1;
  float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ch >= 0) y = *reinterpret_cast<const float4*>(&M.Y[4 * (l16 - ch * qsh)]);
  while (mask) {
    const int b0 = __ffs(mask) - 1;
    mask &= mask - 1;
    const int b1 = mask ? __ffs(mask) - 1 : -1;
    if (b1 >= 0) mask &= mask - 1;
    const int b = upper ? b1 : b0;
    if (b >= 0 && ch >= 0) {
      const int e = base + b;
      const int pos = __float_as_int(M.e2[e].y);
      const float dsel = ch == 0 ? A.a[e].w : (ch == 1 ? A.b[e].x : A.b[e].y);
      atomicAdd(reinterpret_cast<float4*>(gbuf + (size_t)pos * gstride) + 4 + l16,
                make_float4(dsel * y.x, dsel * y.y, dsel * y.z, dsel * y.w));
    }
  }
#endif
}

__device__ __forceinline__ int skip_to(float te, int s, int B, float dt, float t0, float t1) {
  int est = (int)((te - t0) / ((float)B * dt));
  if (est < s + 1) est = s + 1;
  while (fminf(t1, fma_((float)((est + 1) * B), dt, t0)) < te) ++est;
  while (est > s + 1 && fminf(t1, fma_((float)(est * B), dt, t0)) >= te) --est;
  return est;
}

__device__ __forceinline__ void flush_stats(rg_stats* st, const Counters& c, bool hit) {
  const unsigned lane = lane_id();
  // rg_stats fields 0..9, then restarts at field 11 (field 10 = nonfinite_grads)
  const uint32_t v[11] = {lane == 0 ? 1u : 0u, (lane == 0 && hit) ? 1u : 0u, c.slabs, c.pairs,
                          c.evals, c.samples, c.overflows, c.fetches, c.nodes, c.stackov,
                          c.restarts};
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(st);
#pragma unroll
  for (int k = 0; k < 11; ++k) {
    const uint32_t s = __reduce_add_sync(kFull, v[k]);
#ifdef RG_STACK_PROBE
    if (k == 9) {
      if (lane == 0) atomicMax(dst + k, (unsigned long long)c.stackov);
      continue;
    }
#endif
    if (lane == 0 && s) atomicAdd(dst + (k < 10 ? k : k + 1), (unsigned long long)s);
  }
}

// Kahan accumulation
__device__ __forceinline__ void kadd(float& s, float& comp, float x) {
  const float y = x - comp;
  const float t = s + y;
  comp = (t - s) - y;
  s = t;
}

template <class WM>
__device__ __forceinline__ void dbg_put(const RenderArgs& P, int ray, int& dbg_n, int s, int n,
                                        const WM& M, int first) {
  for (int e = (int)lane_id(); e < n; e += 32)
    if (dbg_n + e < P.dbg_cap) {
      int32_t* r = P.dbg_rec + 2 * ((size_t)ray * P.dbg_cap + dbg_n + e);
      r[0] = s;
      r[1] = (int32_t)__float_as_uint(M.e2[first + e].z);
    }
  dbg_n = min(P.dbg_cap, dbg_n + n);
}

// number of held entries with t_entry <= x (the list is sorted by key)
template <int KA, class WM>
__device__ __forceinline__ int held_le(const WM& M, int count, float x) {
  if constexpr (KA == 64) {
    const unsigned m0 = __ballot_sync(kFull, (int)lane_id() < count && M.e0[lane_id()].x <= x);
    const unsigned m1 =
        __ballot_sync(kFull, (int)lane_id() + 32 < count && M.e0[lane_id() + 32].x <= x);
    return __popc(m0) + __popc(m1);
  } else if constexpr (KA <= 128) {
    // independent chunk ballots (a binary search is a chain of dependent loads)
    int n = 0;
#pragma unroll
    for (int h = 0; h < KA / 32; ++h) {
      const int e = 32 * h + (int)lane_id();
      n += __popc(__ballot_sync(kFull, e < count && M.e0[e].x <= x));
    }
    return n;
  } else {
    int lo = 0, len = count;      // warp-uniform binary search (broadcast loads)
    while (len > 0) {
      const int half = len >> 1;
      if (M.e0[lo + half].x <= x) { lo += half + 1; len -= half + 1; } else { len = half; }
    }
    return lo;
  }
}

// INSTR: counters (rg_stats) and the debug dump; the uninstrumented variant
// compiles them out (8 fewer live registers through the march)
template <bool BWD, int GW, bool INSTR, int BASIS, int KA = kA>
__global__ void __launch_bounds__(kBlock, BWD ? RG_MIN_BLOCKS
                                               : (KA == kA ? RG_MIN_BLOCKS_FWD
                                                           : (KA == kAMid ? 4 : 2)))
    k_render(const RenderArgs P) {
  static_assert(KA != kABig || !BWD, "the large-list variant is forward only");
  // dynamic shared memory: per-warp WarpMem (+ WarpAcc in the backward) at fixed
  // offsets; the compiler re-derives the window base (S2R SR_CgaCtaId + LEA) at some
  // loop heads, but the static form measured slower (backward +2.3%)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned lane = lane_id();
  const int wid = threadIdx.x >> 5;
  using WM = std::conditional_t<
      BWD, std::conditional_t<KA == kA, WMBwd, WMBwdMid>,
      std::conditional_t<KA == kA, WMFwd, std::conditional_t<KA == kAMid, WMMid, WMBig>>>;
  WM& M = reinterpret_cast<WM*>(smem_raw)[wid];
  using AC = WarpAccT<WM::kNSlots, BASIS != 0>;
  AC& A = reinterpret_cast<AC*>(smem_raw + sizeof(WM) * kWarps)[BWD ? wid : 0];
  constexpr int kRetK = KA + 32;       // backward: retired (expired, not yet scattered) slots
  int ray;
  Ray R;
  bool inside = true;             // false: a tile-sharding slot outside the rectangle (a miss)
  if (P.cam_mode) {
    const int tile = blockIdx.x;
    if (P.cam.tile > 0) {         // interleaved tile sharding: block = 2x2 pixels of a square
      const int h = P.cam.tile >> 1;
      const int i = tile / (h * h), r = tile - i * (h * h);
      const int lx = 2 * (r % h) + (wid & 1), ly = 2 * (r / h) + (wid >> 1);
      ray = i * P.cam.tile * P.cam.tile + ly * P.cam.tile + lx;
      int px, py;
      inside = camera_tile_pixel(P.cam, ray, px, py);
      camera_ray(P.cam, P.cam.x0 + (inside ? px : 0), P.cam.y0 + (inside ? py : 0), 0.5f, 0.5f,
                 R.o, R.d);
    } else if (P.cam.spp == 1) {  // block = 2x2 pixel tile, warp = pixel
      const int px = 2 * (tile % P.tiles_x) + (wid & 1);
      const int py = 2 * (tile / P.tiles_x) + (wid >> 1);
      if (px >= P.rw || py >= P.rh) return;
      ray = py * P.rw + px;
      camera_ray(P.cam, P.cam.x0 + px, P.cam.y0 + py, 0.5f, 0.5f, R.o, R.d);
    } else {                      // RayGauss4x: block = pixel, warp = one of its 4 subsamples
      const int px = tile % P.rw, py = tile / P.rw;
      ray = tile * 4 + wid;
      camera_ray(P.cam, P.cam.x0 + px, P.cam.y0 + py, sub_off(4, wid & 1), sub_off(4, wid >> 1),
                 R.o, R.d);
    }
  } else {
    ray = blockIdx.x * kWarps + wid;
    if (ray >= P.n_rays) return;
    R.o = make_float3(P.ro[3 * ray], P.ro[3 * ray + 1], P.ro[3 * ray + 2]);
    R.d = make_float3(P.rd[3 * ray], P.rd[3 * ray + 1], P.rd[3 * ray + 2]);
  }
  const rg_config& c = P.c;
  const int B = c.slab_samples;
  const int K = c.hit_capacity;
  const float inv_dt = 1.0f / c.dt;
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, k0c = 0.f, k1c = 0.f, k2c = 0.f;
  float tau = 0.f, tauc = 0.f, T = 1.f;
  int replay = -1;
  Counters cnt = {};
  const bool dbg = INSTR && (!BWD) && P.dbg_rec != nullptr && ray < P.dbg_rays;
  int dbg_n = 0;
  float gr0 = 0.f, gr1 = 0.f, gr2 = 0.f, Pp0 = 0.f, Pp1 = 0.f, Pp2 = 0.f;
  int replay_in = -1;
  int lg0 = -1;   // backward: the ray's log header, loaded with the other per-ray inputs
  if (BWD) {
    gr0 = P.d_rgb[3 * ray]; gr1 = P.d_rgb[3 * ray + 1]; gr2 = P.d_rgb[3 * ray + 2];
    Pp0 = P.rgb_in[3 * ray]; Pp1 = P.rgb_in[3 * ray + 1]; Pp2 = P.rgb_in[3 * ray + 2];
    replay_in = P.replay_in[ray];
    if (P.log) lg0 = P.log[(size_t)ray * kLogWords];
  }
  float t0 = 0.f, t1 = 0.f;
  const bool hit = inside && P.S.n > 0 && clip_exact(P.S.root_box, R.o, R.d, c.t_near, t0, t1);
  if (hit && !(BWD && gr0 == 0.f && gr1 == 0.f && gr2 == 0.f)) {
    R.inv = make_float3(1.0f / R.d.x, 1.0f / R.d.y, 1.0f / R.d.z);
    R.oinv = make_float3(R.o.x * R.inv.x, R.o.y * R.inv.y, R.o.z * R.inv.z);
    {   // Y(d) once per ray (zero past the degree): colour set-up and SH gradients
      float Y[16];
      sh_basis(P.S.deg, R.d.x, R.d.y, R.d.z, Y);
      const int nc = (P.S.deg + 1) * (P.S.deg + 1);
      float ym = 0.f;                 // lane m < nc stores Y_m (register selects, one store)
#pragma unroll
      for (int m = 0; m < 16; ++m) ym = (int)lane == m ? Y[m] : ym;
      if (lane < 16) M.Y[lane] = (int)lane < nc ? ym : 0.f;
      __syncwarp();
    }
    Lanes<GW> L;
    L.j = (int)(lane % GW);
    L.esub = (int)(lane / GW);
    int count = 0, nret = 0;
    unsigned long long cursor = 0;
    bool exhausted = false;
    int32_t* lg = P.log ? P.log + (size_t)ray * kLogWords : nullptr;
    if (lane == 0) {
      M.ls.lp = 1; M.ls.wcur = 0; M.ls.fix = 0;
      M.ls.ok = lg != nullptr && KA != kABig;       // no backward replays the large list
    }
    __syncwarp();
    int& lp = M.ls.lp;
    int& log_ok = M.ls.ok;
    const bool replay_log = BWD && lg != nullptr && lg0 >= 0;
    // stored windows (forward: count so far; backward: how many the forward stored)
    int& nwin = M.ls.nwin;
    int& wlog = M.ls.wl;
    int& wcur = M.ls.wcur;
    int& fix_used = M.ls.fix;   // forward: pair slots used in the ray's own block
    nwin = BWD ? (replay_log ? (lg0 >> 16) : 0) : 0;
    wlog = !BWD && log_ok && RG_STORE_WINDOWS;
    if (lane == 0) M.sst.valid = false;   // forward: persistent traversal restarts on first use
    __syncwarp();
    int nref = 0;                         // forward refills of this ray so far
    // fetch log: the forward appends each query's set-up pair slots [slot0, slot0 + got)
    // (the ray's own pair_fix slots first, then the shared overflow region, one atomic
    // per query) and a (count, arena offset) record; the backward reads them back in
    // the same order (refills and the chunks of slab sets larger than the list)
    auto log_fetch = [&](int got, int slot0) {
      unsigned long long off = 0;
      bool fits = true;
      if (fix_used + got <= P.pair_fix) {
        off = (unsigned long long)ray * P.pair_fix + fix_used;
        fix_used += got;
      } else {
        if (lane == 0 && got > 0) off = atomicAdd(P.arena_ctr, (unsigned long long)got);
        off = shfl64(off, 0) + (unsigned long long)P.n_rays * P.pair_fix;
        fits = (long long)(off + got) <= P.arena_cap;
      }
      if (lp + 2 > kLogWords - nwin && nwin > 0 && lp + 2 <= kLogWords) {
        // fetch records are required, stored windows optional (recomputed by the
        // backward): drop the last stored windows (the stored ones stay a prefix
        // of the ray's windows; no further window is stored)
        nwin = kLogWords - (lp + 2) < nwin ? kLogWords - (lp + 2) : nwin;
        wlog = false;
      }
      if (lp + 2 > kLogWords - nwin || !fits) {
        log_ok = false;
      } else {
        RG_CHECK(lp + 1 < kLogWords - nwin && (long long)(off + got) <= P.arena_cap);
        if (lane == 0) { lg[lp] = got; lg[lp + 1] = (int)off; }
        lp += 2;
        __syncwarp();
        if ((int)lane < got) {
          float4* dst = P.arena + 3 * (off + lane);
          dst[0] = M.e0[slot0 + lane];
          dst[1] = M.e1[slot0 + lane];
          dst[2] = M.e2[slot0 + lane];
        }
      }
    };
    auto read_fetch = [&](int slot0) {
      RG_CHECK(lp + 1 < kLogWords);
      const int got = lg[lp];
      const long long off = (long long)(unsigned)lg[lp + 1];
      RG_CHECK(got >= 0 && got <= 32 && slot0 + got <= WM::kNSlots && off + got <= P.arena_cap);
      lp += 2;
      if ((int)lane < got) {
        const float4* src = P.arena + 3 * (off + lane);
        M.e0[slot0 + lane] = src[0];
        M.e1[slot0 + lane] = src[1];
        M.e2[slot0 + lane] = src[2];
      }
      return got;
    };
    int s = 0;
    while (true) {
      const int k0 = s * B;
      if (!(sample_t(k0, c.dt, t0) < t1)) break;
      const float tlo = fma_((float)k0, c.dt, t0);
      const float thi = fminf(t1, fma_((float)(k0 + B), c.dt, t0));
      // ---- expire Gaussians whose support ended before this slab: chunks of 32
      // slots, compaction from the first expired entry on; the backward first
      // retires the expired pairs (their moments) and scatters them 32 at a time
      {
        int nc = 0;
        bool moved = false;
        auto expire_chunk = [&](int h, int& nc, bool& moved) {
          const int e = 32 * h + (int)lane;
          float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f);
          bool keep = false;
          if (e < count) {
            v0 = M.e0[e];
            keep = !(v0.y < tlo);
          }
          const unsigned km = __ballot_sync(kFull, keep);
          const int nin = min(32, count - 32 * h);
          if (!moved && __popc(km) == nin) { nc += nin; return; }
          moved = true;
          if constexpr (BWD) {   // retire this chunk's expired pairs
            const unsigned gm = __ballot_sync(kFull, e < count && !keep);
            if (nret + __popc(gm) > 32) {
              scatter_batch<BASIS>(P.S, M, A, kRetK, nret >= 32 ? kFull : ((1u << nret) - 1u), R,
                                   P.gbuf, P.gstride);
              nret = 0;
              __syncwarp();
            }
            if ((gm >> lane) & 1u) {
              const int dst = kRetK + nret + __popc(gm & ((1u << lane) - 1u));
              RG_CHECK(dst < WM::kNSlots);
              M.e0[dst] = v0; M.e1[dst] = M.e1[e]; M.e2[dst] = M.e2[e];
              A.a[dst] = A.a[e]; A.b[dst] = A.b[e];
              if (BASIS != 0) A.c[dst] = A.c[e];
            }
            nret += __popc(gm);
            __syncwarp();
          }
          float4 v1 = v0, v2 = v0, a0 = v0;
          float2 a1 = make_float2(0.f, 0.f);
          float a2c = 0.f;
          if (keep) {
            v1 = M.e1[e]; v2 = M.e2[e];
            if (BWD) { a0 = A.a[e]; a1 = A.b[e]; if (BASIS != 0) a2c = A.c[e]; }
          }
          const int dst = nc + __popc(km & ((1u << lane) - 1u));
          __syncwarp();
          if (keep) {
            M.e0[dst] = v0; M.e1[dst] = v1; M.e2[dst] = v2;
            if (BWD) { A.a[dst] = a0; A.b[dst] = a1; if (BASIS != 0) A.c[dst] = a2c; }
          }
          nc += __popc(km);
          __syncwarp();
        };
#pragma unroll
        for (int h = 0; h < (KA == kA ? KA / 32 : 1); ++h) {     // unrolled: the 64-slot list
          if (KA != kA || 32 * h >= count) break;
          expire_chunk(h, nc, moved);
        }
#pragma unroll 1
        for (int h = 0; KA != kA && 32 * h < count; ++h) expire_chunk(h, nc, moved);
        count = nc;
      }
      // 4-slab window (B = 8: 32 samples, one per lane); thr = t_hi of its last slab
      const bool win = (GW == 8) && (B == 8);
      const float thr = win ? fminf(t1, fma_((float)(k0 + 4 * B), c.dt, t0)) : thi;
      // ---- refill in key order until every Gaussian entering by thr is held
      // (large list: when more than K held entries already enter by t_hi, the slab's
      // truncated set -- the K smallest keys -- and its overflow are decided without
      // a query; refills wait until fewer remain, so they come in larger batches)
      while (!exhausted && count < KA && (count == 0 || M.e0[count - 1].x <= thr) &&
             !(KA == kABig && held_le<KA>(M, count, thi) > K)) {
        const int want = min(32, KA - count);
        unsigned long long key = 0;
        uint32_t pos = 0;
        int got;
        if (BWD && replay_log) {      // the forward's set-up pairs: no traversal, no set-up
          got = read_fetch(count);
        } else {
          if constexpr (BWD) {
            got = fetch<WM, !BWD>(P.S, M, R, tlo, t1, cursor, want, key, pos, cnt);
          } else {
            // the first RG_STREAM_FROM refills of a ray by restart queries (most C1 rays
            // need one or two), later ones by the persistent traversal
            if constexpr (!kStream || KA != kA) {
              got = fetch<WM, !BWD>(P.S, M, R, tlo, t1, cursor, want, key, pos, cnt);
            } else {
              if (nref < RG_STREAM_FROM) got = fetch<WM, !BWD>(P.S, M, R, tlo, t1, cursor, want, key, pos, cnt);
              else got = stream_next(P.S, M, R, tlo, t1, cursor, want, key, pos, cnt);
            }
            ++nref;
          }
          if ((int)lane < got) setup_pair<!BWD, BASIS>(P.S, M, count + (int)lane, R, pos);
          if (!BWD && log_ok) log_fetch(got, count);
        }
        if (BWD && (int)lane < got) {
          A.a[count + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
          A.b[count + lane] = make_float2(0.f, 0.f);
          if (BASIS != 0) A.c[count + lane] = 0.f;
        }
        if (lane == 0) cnt.pairs += got;
        count += got;
        if (got < want) exhausted = true;
        __syncwarp();
        if (got > 0) {
          const int l = count - 1;
          cursor = ((unsigned long long)fkey(M.e0[l].x) << 32) | __float_as_uint(M.e2[l].z);
        }
      }
      if (count == 0) break;
      if (M.e0[0].x > thi) {   // empty slab(s): jump to the slab holding the next entry
        s = skip_to(M.e0[0].x, s, B, c.dt, t0, t1);
        continue;
      }
      if (win) {
        // ---- window of slabs s..s+3 when the held list is complete for it and no
        // slab can exceed K: lane k integrates sample 8s + k over all members
        const int n3 = held_le<KA>(M, count, thr);
        if ((n3 < count || exhausted) && n3 <= K) {
          const float tk = sample_t(k0 + (int)lane, c.dt, t0);
          const bool val = tk < t1;
          float sg = 0.f, sr = 0.f, sgg = 0.f, sb = 0.f;
          uint32_t ev = 0;
          // the backward reloads the sums the forward stored for this window
          // (identical values); the instrumented variant recomputes (counters)
          bool stored = false;
          if (BWD && !INSTR) {
            if (wcur < nwin) {
              RG_CHECK(kLogWords - 1 - wcur > 0 && (long long)lg[kLogWords - 1 - wcur] * 32 + 32 <= P.samp_cap);
              const float4 v = P.samp[(size_t)lg[kLogWords - 1 - wcur] * 32 + lane];
              sg = v.x; sr = v.y; sgg = v.z; sb = v.w;
              stored = true;
            }
            ++wcur;
          }
          float2 srg = make_float2(sr, sgg);   // (r, g) sums: one packed FFMA2 per member
#if RG_EVAL_BRANCHFREE
          // predicated form: every lane evaluates, the exact interval test (L2) selects
          if (BASIS == 0) {
#pragma unroll kEvalUnroll
            for (int e = 0; e < (stored ? 0 : n3); ++e) {
              const float4 a = M.e0[e];
              const float4 q = M.e1[e];
              const float cbv = M.e2[e].x;
              const float tau_ = tk - a.z;
              const float wv = ex2_approx(fmaf(tau_, fmaf(q.y, tau_, q.x), a.w));
              const bool in = val && a.x <= tk && tk <= a.y;
              const float w = in ? wv : 0.f;
              sg += w;
              srg = __ffma2_rn(make_float2(w, w), make_float2(q.z, q.w), srg);
              sb = fmaf(w, cbv, sb);
              ev += in ? 1u : 0u;
            }
          } else
#endif
#pragma unroll kEvalUnroll
          for (int e = 0; e < (stored ? 0 : n3); ++e) {
            const float4 a = M.e0[e];
            if (val && a.x <= tk && tk <= a.y) {
              const float4 q = M.e1[e];
              const float cbv = M.e2[e].x;
              const float sge = BASIS != 0 ? M.e2[e].w : 0.f;
              const float tau_ = tk - a.z;
              float qq;
              const float w = basis_w<BASIS>(tau_, a, q, sge, qq);
              sg += w;
              srg = __ffma2_rn(make_float2(w, w), make_float2(q.z, q.w), srg);
              sb = fmaf(w, cbv, sb);
              ++ev;
            }
          }
          sr = srg.x;
          sgg = srg.y;
          if (!BWD && wlog && log_ok) {   // store this window's sums for the backward
            unsigned long long off = 0;
            if (lane == 0) off = atomicAdd(P.samp_ctr, 32ull);
            off = shfl64(off, 0);
            // keep >= 8 record words for later fetch records (they have priority)
            if (kLogWords - nwin - lp < 9 || (long long)(off + 32) > P.samp_cap) {
              wlog = false;
            } else {
              RG_CHECK(kLogWords - 1 - nwin > lp);
              if (lane == 0) lg[kLogWords - 1 - nwin] = (int)(off >> 5);
              P.samp[off + lane] = make_float4(sg, sr, sgg, sb);
              ++nwin;
            }
          }
          const bool live0 = val && sg > 0.f;
          const float x = live0 ? sg * c.dt : 0.f;
          float incl = x;
#pragma unroll
          for (int dd = 1; dd < 32; dd <<= 1) {
            const float v = __shfl_up_sync(kFull, incl, dd);
            if ((int)lane >= dd) incl += v;
          }
          const float Tb = ex2_approx(-(tau + (incl - x)) * kLog2e);
          const float e_s = ex2_approx(-x * kLog2e);
          const float al = alpha_of(x, e_s);
          // value path (never a decision): MUFU reciprocal, ~1 ulp, no IEEE-division slow path
          const float inv_s = live0 ? __fdividef(1.0f, sg) : 0.f;
          const float cr = sr * inv_s, cg = sgg * inv_s, cb = sb * inv_s;
          const float wgt = live0 ? Tb * al : 0.f;
          float p0 = wgt * cr, p1 = wgt * cg, p2 = wgt * cb;
#pragma unroll
          for (int dd = 1; dd < 32; dd <<= 1) {
            const float v0 = __shfl_up_sync(kFull, p0, dd);
            const float v1 = __shfl_up_sync(kFull, p1, dd);
            const float v2 = __shfl_up_sync(kFull, p2, dd);
            if ((int)lane >= dd) { p0 += v0; p1 += v1; p2 += v2; }
          }
          // first slab whose end has T <= T_eps (forward) / the recorded one (backward)
          int wlast = 3;
          bool term = false;
          if (BWD) {
            if (replay_in >= s && replay_in <= s + 3) { wlast = replay_in - s; term = true; }
          } else {
            const float Te = ex2_approx(-(tau + incl) * kLog2e);
            const unsigned tm = __ballot_sync(kFull, ((lane & 7u) == 7u) && Te <= c.t_eps);
            if (tm) { wlast = (__ffs(tm) - 1) >> 3; term = true; }
          }
          const int last = 8 * wlast + 7;
          const bool inwin = (int)lane <= last;
          const bool live = live0 && inwin;
          // per-slab sets (counters, debug dump): members of slab s+w, key order
          for (int w = 0; w <= wlast && INSTR && (P.stats != nullptr || dbg); ++w) {
            const float lo_w = fma_((float)(k0 + 8 * w), c.dt, t0);
            if (!(sample_t(k0 + 8 * w, c.dt, t0) < t1)) break;
            const float hi_w = fminf(t1, fma_((float)(k0 + 8 * w + 8), c.dt, t0));
            bool any_w = false;
            for (int h = 0; 32 * h < n3; ++h) {
              const int e = 32 * h + (int)lane;
              const unsigned qm = __ballot_sync(
                  kFull, e < n3 && M.e0[e].x <= hi_w && M.e0[e].y >= lo_w);
              any_w |= qm != 0u;
              if (dbg && qm) {
                if ((qm >> lane) & 1u) {
                  const int r = dbg_n + __popc(qm & ((1u << lane) - 1u));
                  if (r < P.dbg_cap) {
                    int32_t* rr = P.dbg_rec + 2 * ((size_t)ray * P.dbg_cap + r);
                    rr[0] = s + w;
                    rr[1] = (int32_t)__float_as_uint(M.e2[e].z);
                  }
                }
                dbg_n = min(P.dbg_cap, dbg_n + __popc(qm));
              }
            }
            if (any_w && lane == 0) cnt.slabs++;
          }
          {
            const uint32_t evs = __reduce_add_sync(kFull, inwin ? ev : 0u);
            const unsigned smask = __ballot_sync(kFull, live);
            if (lane == 0) { cnt.evals += evs; cnt.samples += __popc(smask); }
          }
          if (BWD) {
            SampleGrad H = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (live) {
              const float Ta = Tb * e_s;
              H.dc0 = gr0 * wgt; H.dc1 = gr1 * wgt; H.dc2 = gr2 * wgt;
              const float gcj = gr0 * cr + gr1 * cg + gr2 * cb;
              const float gS =
                  gr0 * (Pp0 - (C0 + p0)) + gr1 * (Pp1 - (C1 + p1)) + gr2 * (Pp2 - (C2 + p2));
              H.dls = c.dt * (Ta * gcj - gS);
              H.gc = H.dc0 * cr + H.dc1 * cg + H.dc2 * cb;
              H.inv = inv_s;
            }
            // dL/dw_e = (dls - gc/sigma) + <dc, c_e>/sigma: per-sample coefficients
            // (zero for dead samples, so the member loop needs no liveness test)
            A.s0[lane] = make_float4(tk, H.dls - H.gc * H.inv, H.dc0 * H.inv, H.dc1 * H.inv);
            A.s1[lane] = H.dc2 * H.inv;
            __syncwarp();
            // lane = (member, part): P2 members per pass, each member's window samples
            // split into 32/P2 parts of P2 samples; parts reduced by xor shuffles
            const int P2 = (RG_P2_MIN <= 4 && n3 <= 4) ? 4 : (n3 <= 8 ? 8 : (n3 <= 16 ? 16 : 32));
            for (int base = 0; base < n3; base += P2) {
              const int e = base + ((int)lane & (P2 - 1));
              const int part0 = (int)lane & ~(P2 - 1);   // first sample of this lane's part
              float a0 = 0.f, a1 = 0.f, a2 = 0.f, a5 = 0.f, a6 = 0.f;
              float2 a34 = make_float2(0.f, 0.f);   // (dc_r, dc_g) moments: packed FFMA2
              float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
              if (e < n3) {
                a = M.e0[e];
                const float4 q = M.e1[e];
                const float cbv = M.e2[e].x;
                const float sge = BASIS != 0 ? M.e2[e].w : 0.f;
                // conservative sample range (+-1; the exact test below decides): a
                // reciprocal multiply, not two IEEE divisions per member and window
                const float kf = (float)k0 + 0.5f;
                int kl = (int)floorf((a.x - t0) * inv_dt - kf) - 1;
                int kh = (int)ceilf((a.y - t0) * inv_dt - kf) + 1;
                kl = max(kl, part0);
                kh = min(kh, min(last, part0 + P2 - 1));
#if RG_GRAD_BRANCHFREE
                if (BASIS == 0) {
#if RG_GRAD_FIXED
                  // the whole part, a fixed trip count: samples outside the support or
                  // past the termination carry zero coefficients (A.s0 / A.s1) or fail
                  // the interval test, so they add exactly nothing
                  (void)kl; (void)kh;
#pragma unroll 4
                  for (int k = part0; k < part0 + P2; ++k) {
#else
#pragma unroll kMemberUnroll
                  for (int k = kl; k <= kh; ++k) {
#endif
                    const float4 s0 = A.s0[k];
                    const float tkk = s0.x;
                    const float b2 = A.s1[k];
                    const float tau_ = tkk - a.z;
                    const float wv = ex2_approx(fmaf(tau_, fmaf(q.y, tau_, q.x), a.w));
                    const float w = (a.x <= tkk && tkk <= a.y) ? wv : 0.f;
                    const float dldw = fmaf(s0.z, q.z, fmaf(s0.w, q.w, fmaf(b2, cbv, s0.y)));
                    const float wd = w * dldw;
                    a0 += wd;
                    a1 = fmaf(wd, tau_, a1);
                    a2 = fmaf(wd * tau_, tau_, a2);
                    a34 = __ffma2_rn(make_float2(w, w), make_float2(s0.z, s0.w), a34);
                    a5 = fmaf(w, b2, a5);
                  }
                } else
#endif
#pragma unroll kMemberUnroll
                for (int k = kl; k <= kh; ++k) {
                  const float4 s0 = A.s0[k];
                  const float tkk = s0.x;
                  if (a.x <= tkk && tkk <= a.y) {
                    const float b2 = A.s1[k];
                    const float tau_ = tkk - a.z;
                    float qq;
                    const float w = basis_w<BASIS>(tau_, a, q, sge, qq);
                    const float dldw = fmaf(s0.z, q.z, fmaf(s0.w, q.w, fmaf(b2, cbv, s0.y)));
                    const float wd = basis_psi<BASIS>(w, qq, sge) * dldw;
                    a0 += wd;
                    a1 = fmaf(wd, tau_, a1);
                    a2 = fmaf(wd * tau_, tau_, a2);
                    a34 = __ffma2_rn(make_float2(w, w), make_float2(s0.z, s0.w), a34);
                    a5 = fmaf(w, b2, a5);
                    if (BASIS != 0) a6 = fmaf(w, dldw, a6);
                  }
                }
              }
              float a3 = a34.x, a4 = a34.y;
              for (int off = P2; off < 32; off <<= 1) {
                a0 += __shfl_xor_sync(kFull, a0, off);
                a1 += __shfl_xor_sync(kFull, a1, off);
                a2 += __shfl_xor_sync(kFull, a2, off);
                a3 += __shfl_xor_sync(kFull, a3, off);
                a4 += __shfl_xor_sync(kFull, a4, off);
                a5 += __shfl_xor_sync(kFull, a5, off);
                if (BASIS != 0) a6 += __shfl_xor_sync(kFull, a6, off);
              }
              if (e < n3 && part0 == 0) {
                float4 v = A.a[e];
                float2 w2 = A.b[e];
                v.x += a0; v.y += a1; v.z += a2; v.w += a3;
                w2.x += a4; w2.y += a5;
                A.a[e] = v;
                A.b[e] = w2;
                if (BASIS != 0) A.c[e] += a6;
              }
            }
            __syncwarp();
          }
          kadd(tau, tauc, __shfl_sync(kFull, incl, last));
          kadd(C0, k0c, __shfl_sync(kFull, p0, last));
          kadd(C1, k1c, __shfl_sync(kFull, p1, last));
          kadd(C2, k2c, __shfl_sync(kFull, p2, last));
          T = ex2_approx(-tau * kLog2e);
          if (term) {
            if (!BWD) replay = s + wlast;
            break;
          }
          s += 4;
          continue;
        }
      }
      const int n_in = held_le<KA>(M, count, thi);
      const int n_use = min(n_in, K);
      const bool more = (n_in == KA) && !exhausted && (K > KA);
      if (n_in > K) {
        if (lane == 0) cnt.overflows++;
      } else if (INSTR && !BWD && n_in == K && n_in == KA && !exhausted) {   // counter only
        unsigned long long pk;
        uint32_t pp;
        if (fetch<WM, !BWD>(P.S, M, R, tlo, thi, cursor, 1, pk, pp, cnt) > 0 && lane == 0) cnt.overflows++;
      }
      if (!BWD && (more || (INSTR && n_in == K && n_in == KA && !exhausted))) {
        __syncwarp();                        // a restart query reused the traversal memory
        if (lane == 0) M.sst.valid = false;
        __syncwarp();
      }
      if (dbg) dbg_put(P, ray, dbg_n, s, n_use, M, 0);
      for (int g0 = 0; g0 < B; g0 += GW) {
        const float tk = sample_t(k0 + g0 + L.j, c.dt, t0);
        const bool val = (g0 + L.j < B) && (tk < t1);
        float sg = 0.f, sr = 0.f, sgg = 0.f, sb = 0.f;
        uint32_t ev = 0;
        eval_range<GW, BASIS, BWD>(M, 0, n_use, L, tk, val, sg, sr, sgg, sb, ev);
        if (more) {   // slab set larger than the active list: stream the rest
          unsigned long long cur2 = cursor;
          int remaining = K - n_use;
          bool full_last = true;
          while (remaining > 0) {
            const int want = min(32, remaining);
            unsigned long long key;
            uint32_t pos;
            const int got = fetch<WM, !BWD>(P.S, M, R, tlo, thi, cur2, want, key, pos, cnt);
            if ((int)lane < got) setup_pair<!BWD, BASIS>(P.S, M, KA + (int)lane, R, pos);
            __syncwarp();
            if (!BWD && log_ok) log_fetch(got, KA);
            eval_range<GW, BASIS, BWD>(M, KA, KA + got, L, tk, val, sg, sr, sgg, sb, ev);
            if (dbg && g0 == 0) dbg_put(P, ray, dbg_n, s, got, M, KA);
            if (g0 == 0 && lane == 0) cnt.pairs += got;
            remaining -= got;
            if (got > 0) cur2 = shfl64(key, got - 1);
            __syncwarp();
            if (got < want) { full_last = false; break; }
          }
          if (INSTR && g0 == 0 && remaining == 0 && full_last) {   // overflow counter only
            unsigned long long pk;
            uint32_t pp;
            if (fetch<WM, !BWD>(P.S, M, R, tlo, thi, cur2, 1, pk, pp, cnt) > 0 && lane == 0) cnt.overflows++;
          }
        }
        cnt.evals += ev;
        // reduce over the entry subsets: every lane of sample j holds the totals
#pragma unroll
        for (int off = GW; off < 32; off <<= 1) {
          sg += __shfl_xor_sync(kFull, sg, off);
          sr += __shfl_xor_sync(kFull, sr, off);
          sgg += __shfl_xor_sync(kFull, sgg, off);
          sb += __shfl_xor_sync(kFull, sb, off);
        }
        // ---- composite the group front to back (Eq. 4): segmented scans over GW lanes
        const bool live = val && sg > 0.f;
        const float x = live ? sg * c.dt : 0.f;
        float incl = x;
#pragma unroll
        for (int dd = 1; dd < GW; dd <<= 1) {
          const float v = __shfl_up_sync(kFull, incl, dd, GW);
          if (L.j >= dd) incl += v;
        }
        const float excl = incl - x;
        const float Tb = ex2_approx(-(tau + excl) * kLog2e);   // T before this sample
        const float e_s = ex2_approx(-x * kLog2e);
        const float al = alpha_of(x, e_s);
        const float inv_s = live ? __fdividef(1.0f, sg) : 0.f;
        const float cr = sr * inv_s, cg = sgg * inv_s, cb = sb * inv_s;
        const float wgt = live ? Tb * al : 0.f;
        float p0 = wgt * cr, p1 = wgt * cg, p2 = wgt * cb;
#pragma unroll
        for (int dd = 1; dd < GW; dd <<= 1) {
          const float v0 = __shfl_up_sync(kFull, p0, dd, GW);
          const float v1 = __shfl_up_sync(kFull, p1, dd, GW);
          const float v2 = __shfl_up_sync(kFull, p2, dd, GW);
          if (L.j >= dd) { p0 += v0; p1 += v1; p2 += v2; }
        }
        if (BWD) {   // per-sample dL/dsigma_k, dL/dc_k for the gradient pass
          SampleGrad H = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          if (live) {
            const float Ta = Tb * e_s;
            H.dc0 = gr0 * wgt; H.dc1 = gr1 * wgt; H.dc2 = gr2 * wgt;
            const float gcj = gr0 * cr + gr1 * cg + gr2 * cb;
            const float gS =
                gr0 * (Pp0 - (C0 + p0)) + gr1 * (Pp1 - (C1 + p1)) + gr2 * (Pp2 - (C2 + p2));
            H.dls = c.dt * (Ta * gcj - gS);
            H.gc = H.dc0 * cr + H.dc1 * cg + H.dc2 * cb;
            H.inv = inv_s;
          }
          if (L.esub == 0) {
            A.s0[L.j] = make_float4(tk, H.dls - H.gc * H.inv, H.dc0 * H.inv, H.dc1 * H.inv);
            A.s1[L.j] = H.dc2 * H.inv;
          }
        }
        const float tot_x = __shfl_sync(kFull, incl, GW - 1, GW);
        const float t0c = __shfl_sync(kFull, p0, GW - 1, GW);
        const float t1c = __shfl_sync(kFull, p1, GW - 1, GW);
        const float t2c = __shfl_sync(kFull, p2, GW - 1, GW);
        kadd(tau, tauc, tot_x);
        kadd(C0, k0c, t0c);
        kadd(C1, k1c, t1c);
        kadd(C2, k2c, t2c);
        T = ex2_approx(-tau * kLog2e);
        const unsigned smask = __ballot_sync(kFull, live && L.esub == 0);
        if (lane == 0) cnt.samples += __popc(smask);
        if (BWD) {
          grad_range<GW, BASIS>(M, A, 0, n_use);
          if (more) {
            unsigned long long cur2 = cursor;
            int remaining = K - n_use;
            while (remaining > 0) {
              const int want = min(32, remaining);
              unsigned long long key;
              uint32_t pos;
              int got;
              if (replay_log) {           // the forward logged this chunk's set-up pairs
                got = read_fetch(KA);
              } else {
                got = fetch<WM, !BWD>(P.S, M, R, tlo, thi, cur2, want, key, pos, cnt);
                if ((int)lane < got) setup_pair<!BWD, BASIS>(P.S, M, KA + (int)lane, R, pos);
              }
              if ((int)lane < got) {
                A.a[KA + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                A.b[KA + lane] = make_float2(0.f, 0.f);
                if (BASIS != 0) A.c[KA + lane] = 0.f;
              }
              __syncwarp();
              grad_range<GW, BASIS>(M, A, KA, KA + got);
              scatter_batch<BASIS>(P.S, M, A, KA, got >= 32 ? kFull : ((1u << got) - 1u), R, P.gbuf,
                            P.gstride);
              remaining -= got;
              if (got > 0) {
                const int l = KA + got - 1;
                cur2 = replay_log ? (((unsigned long long)fkey(M.e0[l].x) << 32) | __float_as_uint(M.e2[l].z))
                                  : shfl64(key, got - 1);
              }
              __syncwarp();
              if (got < want) break;
            }
          }
        }
      }
      if (lane == 0) cnt.slabs++;
      if (BWD) {
        if (s == replay_in) break;
      } else if (T <= c.t_eps) {
        replay = s;
        break;
      }
      ++s;
    }
    if (BWD) {
#pragma unroll 1
      for (int h = 0; 32 * h < count; ++h) {    // the pairs still held, 32 at a time
        const int c = count - 32 * h;
        scatter_batch<BASIS>(P.S, M, A, 32 * h, c >= 32 ? kFull : ((1u << c) - 1u), R, P.gbuf,
                             P.gstride);
      }
      scatter_batch<BASIS>(P.S, M, A, kRetK, nret >= 32 ? kFull : ((1u << nret) - 1u), R, P.gbuf,
                    P.gstride);
    } else if (lg != nullptr && lane == 0) {
      lg[0] = log_ok ? (lp | (nwin << 16)) : -1;
    }
  }
  if (!BWD && lane == 0) {
    P.rgb[3 * ray] = C0 + T * c.background[0];
    P.rgb[3 * ray + 1] = C1 + T * c.background[1];
    P.rgb[3 * ray + 2] = C2 + T * c.background[2];
    P.T[ray] = T;
    P.replay[ray] = replay;
    if (INSTR && P.dbg_counts && ray < P.dbg_rays) P.dbg_counts[ray] = dbg_n;
  }
  if (INSTR && P.stats) flush_stats(P.stats, cnt, hit);
}

// (mu, M) -> (mu, q, s) and Morton -> caller order
__global__ void __launch_bounds__(256) k_finalize(const float* gbuf, int gstride,
                                                  const uint32_t* order, rg_gaussians g,
                                                  rg_gaussian_grads out, rg_stats* stats) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.n) return;
  const int i = (int)order[p];
  const float* row = gbuf + (size_t)p * gstride;
  const float* q = g.quat + 4 * (size_t)i;
  const float* s = g.scale + 3 * (size_t)i;
  const float w = q[0], x = q[1], y = q[2], z = q[3];
  const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                      2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                      2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
  float dR[9];
  float ds[3];
  // a row that received no geometry gradient (never hit: e.g. an inactive, possibly
  // non-finite, Gaussian) converts to exact zeros, not 0 * NaN
  bool any = false;
  for (int k = 0; k < 10; ++k) any |= (k != 3) && row[k] != 0.f;
  // the backward accumulates v = sum (Sw x' + Sw1 d) and the symmetric
  // S = sum (Sw x'x'^T + Sw1 (x'd^T + d x'^T) + Sw2 d d^T) (scatter_batch):
  // dL/dmu = M^T M v, dL/dM = -M S, with M_ab = R_ba / s_a
  float Mx[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Mx[3 * a + b] = R[3 * b + a] / s[a];
  const float Sm[9] = {row[4], row[5], row[6], row[5], row[7], row[8], row[6], row[8], row[9]};
  float gmu[3] = {0.f, 0.f, 0.f};
  if (any) {
    float mv[3];
    for (int a = 0; a < 3; ++a) mv[a] = Mx[3 * a] * row[0] + Mx[3 * a + 1] * row[1] + Mx[3 * a + 2] * row[2];
    for (int b = 0; b < 3; ++b) gmu[b] = Mx[b] * mv[0] + Mx[3 + b] * mv[1] + Mx[6 + b] * mv[2];
  }
  for (int a = 0; a < 3; ++a) {
    ds[a] = 0.f;
    for (int b = 0; b < 3; ++b) {
      // dL/dM_ab = -(M S)_ab
      const float dM = any ? -(Mx[3 * a] * Sm[b] + Mx[3 * a + 1] * Sm[3 + b] + Mx[3 * a + 2] * Sm[6 + b])
                           : 0.f;
      ds[a] -= any ? dM * R[3 * b + a] / (s[a] * s[a]) : 0.f;
      dR[3 * b + a] = any ? dM / s[a] : 0.f;
    }
  }
  // d R / d q (polynomial ARITH-1 differentiated)
  float dq[4];
  dq[0] = dR[1] * (-2 * z) + dR[2] * (2 * y) + dR[3] * (2 * z) + dR[5] * (-2 * x) +
          dR[6] * (-2 * y) + dR[7] * (2 * x);
  dq[1] = dR[1] * (2 * y) + dR[2] * (2 * z) + dR[3] * (2 * y) + dR[4] * (-4 * x) +
          dR[5] * (-2 * w) + dR[6] * (2 * z) + dR[7] * (2 * w) + dR[8] * (-4 * x);
  dq[2] = dR[0] * (-4 * y) + dR[1] * (2 * x) + dR[2] * (2 * w) + dR[3] * (2 * x) +
          dR[5] * (2 * z) + dR[6] * (-2 * w) + dR[7] * (2 * z) + dR[8] * (-4 * y);
  dq[3] = dR[0] * (-4 * z) + dR[1] * (-2 * w) + dR[2] * (2 * x) + dR[3] * (2 * w) +
          dR[4] * (-4 * z) + dR[5] * (2 * y) + dR[6] * (2 * x) + dR[7] * (2 * y);
  if (!any) dq[0] = dq[1] = dq[2] = dq[3] = 0.f;
  uint32_t bad = 0;
  auto put = [&](float* base, size_t k, float v) {
    if (!isfinite(v)) ++bad;
    if (base) base[k] += v;
  };
  for (int a = 0; a < 3; ++a) put(out.mean, 3 * (size_t)i + a, gmu[a]);
  put(out.density, i, row[3]);
  for (int a = 0; a < 3; ++a) put(out.scale, 3 * (size_t)i + a, ds[a]);
  for (int a = 0; a < 4; ++a) put(out.quat, 4 * (size_t)i + a, dq[a]);
  if (bad && stats) atomicAdd(&stats->nonfinite_grads, (unsigned long long)bad);
}

// appearance part of the rows, one warp per Gaussian, coalesced on the caller
// layout: SH grads from channel-major [3][ncp], SG from lobe-major [G][8]
__global__ void __launch_bounds__(256) k_finalize_app(const float* gbuf, int gstride,
                                                      const uint32_t* order, rg_gaussians g,
                                                      rg_gaussian_grads out, rg_stats* stats) {
  const int lane = threadIdx.x & 31;
  const int nc = (g.sh_degree + 1) * (g.sh_degree + 1), nc3 = 3 * nc;
  const int ncp = sh_pad(g.sh_degree), G = g.sg_count;
  uint32_t bad = 0;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < g.n;
       p += (gridDim.x * blockDim.x) >> 5) {
    const size_t i = order[p];
    const float* ap = gbuf + (size_t)p * gstride + 16;
    // <= 97 values per row: up to 4 per lane, every load issued before the first use
    // (the per-element read-modify-write chain was latency-bound)
    constexpr int kPer = (3 * 16 + 7 * 7 + 31) / 32;
    float v[kPer], o[kPer];
    float* dst[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int f = lane + 32 * t;
      dst[t] = nullptr;
      v[t] = 0.f;
      if (f < nc3) {
        const int m = f / 3, ch = f - 3 * m;
        v[t] = ap[ch * ncp + m];
        if (out.sh) dst[t] = out.sh + i * nc3 + f;
      } else if (f < nc3 + 7 * G) {
        const int j = (f - nc3) / 7, r = (f - nc3) - 7 * j;
        v[t] = ap[3 * ncp + 8 * j + r];
        const size_t ij = i * G + j;
        if (r < 3) dst[t] = out.sg_amp ? out.sg_amp + 3 * ij + r : nullptr;
        else if (r == 3) dst[t] = out.sg_sharp ? out.sg_sharp + ij : nullptr;
        else dst[t] = out.sg_axis ? out.sg_axis + 3 * ij + r - 4 : nullptr;
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) o[t] = dst[t] ? *dst[t] : 0.f;
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      bad += !isfinite(v[t]);
      if (dst[t]) *dst[t] = o[t] + v[t];
    }
  }
  bad = __reduce_add_sync(0xffffffffu, bad);
  if (bad && lane == 0 && stats) atomicAdd(&stats->nonfinite_grads, (unsigned long long)bad);
}

__global__ void k_camera_rays(const rg_camera cam, float* o, float* d, int64_t n) {
  const int rw = cam.x1 - cam.x0;
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  float3 oo = make_float3(0.f, 0.f, 0.f), dd = oo;
  if (cam.tile > 0) {
    int px, py;
    if (camera_tile_pixel(cam, r, px, py))
      camera_ray(cam, cam.x0 + px, cam.y0 + py, 0.5f, 0.5f, oo, dd);
  } else {
    const int64_t pix = r / cam.spp;
    const int s = (int)(r - pix * cam.spp);
    camera_ray(cam, cam.x0 + (int)(pix % rw), cam.y0 + (int)(pix / rw), sub_off(cam.spp, s & 1),
               sub_off(cam.spp, s >> 1), oo, dd);
  }
  o[3 * r] = oo.x; o[3 * r + 1] = oo.y; o[3 * r + 2] = oo.z;
  d[3 * r] = dd.x; d[3 * r + 1] = dd.y; d[3 * r + 2] = dd.z;
}

__global__ void k_l1(const float* a, const float* b, int64_t n, float scale, float* g,
                     float* loss) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float diff = a[i] - b[i];
    g[i] = diff > 0.f ? scale : (diff < 0.f ? -scale : 0.f);
    acc += fabsf(diff);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(loss, acc * scale);
}

SceneView view_of(const rg_bvh& b) {
  SceneView S;
  S.geom = reinterpret_cast<const float4*>(b.geom);
  S.app = b.app;
  S.nodes = reinterpret_cast<const float4*>(b.nodes);
  S.wide = reinterpret_cast<const WideNode*>(b.wide);
  S.root_box = b.root_box;
  S.n = b.n;
  S.deg = b.sh_degree;
  S.lobes = b.sg_count;
  S.app_stride = b.app_stride;
  return S;
}

void ray_grid(RenderArgs& A, const rg_rays* rays, const rg_camera* cam, dim3& grid) {
  if (cam) {
    A.cam_mode = 1;
    A.cam = *cam;
    A.rw = cam->x1 - cam->x0;
    A.rh = cam->y1 - cam->y0;
    A.n_rays = (int)camera_ray_slots(*cam);
    A.tiles_x = (A.rw + 1) / 2;
    if (cam->tile > 0)            // owned squares x (tile/2)^2 blocks of 2x2 pixels
      grid = dim3((unsigned)(camera_owned_squares(*cam) * (cam->tile / 2) * (cam->tile / 2)));
    else
      grid = cam->spp == 1 ? dim3((unsigned)(A.tiles_x * ((A.rh + 1) / 2)))
                           : dim3((unsigned)(A.rw * A.rh));   // spp = 4: one block per pixel
  } else {
    A.cam_mode = 0;
    A.ro = rays->origin;
    A.rd = rays->dir;
    A.n_rays = rays->n;
    grid = dim3((unsigned)((rays->n + kWarps - 1) / kWarps));
  }
}

// dynamic shared memory above the 48 KB default needs a per-kernel opt-in
template <bool BWD, int GW, bool INSTR, int BASIS, int KA = kA>
void launch_one(const RenderArgs& A, dim3 grid, size_t smem, cudaStream_t st) {
  static bool opted = false;
  if (!opted) {
    cudaFuncSetAttribute(k_render<BWD, GW, INSTR, BASIS, KA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    opted = true;
  }
  k_render<BWD, GW, INSTR, BASIS, KA><<<grid, kBlock, smem, st>>>(A);
}

template <bool BWD, int GW, int BASIS>
void launch_gw(const RenderArgs& A, dim3 grid, size_t smem, cudaStream_t st) {
  if (A.stats != nullptr || A.dbg_rec != nullptr) launch_one<BWD, GW, true, BASIS>(A, grid, smem, st);
  else launch_one<BWD, GW, false, BASIS>(A, grid, smem, st);
}

constexpr size_t kSmemFwd = sizeof(WMFwd) * kWarps;
constexpr size_t kSmemBwd = (sizeof(WMBwd) + sizeof(WarpAccT<WMBwd::kNSlots>)) * kWarps;
constexpr size_t kSmemBwdG = (sizeof(WMBwd) + sizeof(WarpAccT<WMBwd::kNSlots, false>)) * kWarps;
constexpr size_t kSmemBwdMid = (sizeof(WMBwdMid) + sizeof(WarpAccT<WMBwdMid::kNSlots>)) * kWarps;
// the Gaussian backward (no per-slot c) fits RG_MIN_BLOCKS (4) blocks per SM; 5 blocks
// (96 registers) measured slower, 4.83 -> 5.38 ms (profiles/r2/ab_bwd_blocks.log)
static_assert(RG_MIN_BLOCKS * (kSmemBwdG + 1024) <= 228 * 1024, "backward blocks per SM");
// 4 resident backward blocks must fit the 196 KB shared-memory carve-out (1 KB
// reserved per block): a larger carve-out halves L1 and costs ~6% (measured)
static_assert(kSmemBwd <= 48 * 1024 + 128, "backward block exceeds the 196 KB carve-out budget");
constexpr size_t kSmemBig = sizeof(WMBig) * kWarps;
constexpr size_t kSmemMid = sizeof(WMMid) * kWarps;
static_assert(2 * (kSmemBig + 1024) <= 228 * 1024, "two large-list blocks per SM");

template <bool BWD>
void launch_render(const RenderArgs& A, dim3 grid, size_t smem, cudaStream_t st) {
  const int B = A.c.slab_samples;
  if (BWD && A.c.basis == 0) smem = kSmemBwdG;   // the Gaussian backward has no per-slot c
  // forward large-list variant (rg_config.list_capacity, Gaussian basis, B >= 5)
  if constexpr (!BWD) {
    const bool instr = A.stats != nullptr || A.dbg_rec != nullptr;
    if (A.c.list_capacity > kAMid && A.c.basis == 0 && B >= 5 && A.c.hit_capacity < kABig) {
      if (instr) launch_one<false, 8, true, 0, kABig>(A, grid, kSmemBig, st);
      else launch_one<false, 8, false, 0, kABig>(A, grid, kSmemBig, st);
      return;
    }
    if (A.c.list_capacity > kA && A.c.basis == 0 && B >= 5) {
      if (instr) launch_one<false, 8, true, 0, kAMid>(A, grid, kSmemMid, st);
      else launch_one<false, 8, false, 0, kAMid>(A, grid, kSmemMid, st);
      return;
    }
  } else {
    // the backward replays the forward's log, so it runs the same list: the medium
    // list has a backward variant; the large list's forward writes no log (its rays
    // are re-traversed by the 64-slot backward)
    if (A.c.list_capacity > kA && A.c.list_capacity <= kAMid && A.c.basis == 0 && B >= 5) {
      if (A.stats != nullptr) launch_one<true, 8, true, 0, kAMid>(A, grid, kSmemBwdMid, st);
      else launch_one<true, 8, false, 0, kAMid>(A, grid, kSmemBwdMid, st);
      return;
    }
  }
  // non-Gaussian bases (NEXT-3) are instantiated for GW = 8 only (B >= 5; the API
  // rejects them otherwise)
  if (B >= 5) {
    switch (A.c.basis) {
      case 1: launch_gw<BWD, 8, 1>(A, grid, smem, st); break;
      case 2: launch_gw<BWD, 8, 2>(A, grid, smem, st); break;
      case 3: launch_gw<BWD, 8, 3>(A, grid, smem, st); break;
      case 4: launch_gw<BWD, 8, 4>(A, grid, smem, st); break;
      case 5: launch_gw<BWD, 8, 5>(A, grid, smem, st); break;
      default: launch_gw<BWD, 8, 0>(A, grid, smem, st);
    }
  } else if (B >= 3) launch_gw<BWD, 4, 0>(A, grid, smem, st);
  else if (B == 2) launch_gw<BWD, 2, 0>(A, grid, smem, st);
  else launch_gw<BWD, 1, 0>(A, grid, smem, st);
}



// fetch-log layout (rg_internal.cuh): counter | per-ray records | arena
void set_log(RenderArgs& A, const void* log, size_t log_bytes, int n_rays) {
  if (!log) return;
  char* base = const_cast<char*>(static_cast<const char*>(log));
  const size_t hdr = fetch_log_header_bytes(n_rays);
  A.arena_ctr = reinterpret_cast<unsigned long long*>(base);
  A.log = reinterpret_cast<int32_t*>(base + 256);
  A.arena = reinterpret_cast<float4*>(base + hdr);
  const size_t rest = log_bytes - hdr;
  A.arena_cap = (long long)(rest / 80);
  // per-ray blocks of 32 slots (a ray's first fetch always fits) when the arena has
  // >= 48 per ray (the default budget); later fetches use the shared region
  A.pair_fix = A.arena_cap >= 48ll * n_rays ? 32 : 0;
  A.samp_ctr = reinterpret_cast<unsigned long long*>(base + 8);
  A.samp = reinterpret_cast<float4*>(base + hdr + 48 * (size_t)A.arena_cap);
  A.samp_cap = (long long)((rest - 48 * (size_t)A.arena_cap) / 16);
}

}  // namespace

cudaError_t launch_camera_rays(const rg_camera& cam, float* o, float* d, cudaStream_t st) {
  const int64_t n = camera_ray_slots(cam);
  if (n > 0) {
    k_camera_rays<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cam, o, d, n);
    count_launches(1);
  }
  return cudaGetLastError();
}

cudaError_t launch_forward(const rg_gaussians& g, const rg_bvh& b, const rg_config& c,
                           const rg_rays* rays, const rg_camera* cam, float* rgb, float* T,
                           int32_t* replay, void* log, size_t log_bytes, rg_stats* stats,
                           int dbg_rays, int dbg_cap, int32_t* dbg_counts, int32_t* dbg_rec,
                           cudaStream_t st) {
  (void)g;
  RenderArgs A = {};
  A.S = view_of(b);
  A.c = c;
  dim3 grid;
  ray_grid(A, rays, cam, grid);
  if (A.n_rays == 0) return cudaSuccess;
  A.rgb = rgb; A.T = T; A.replay = replay; A.stats = stats;
  set_log(A, log, log_bytes, A.n_rays);
  if (log) cudaMemsetAsync(A.arena_ctr, 0, 16, st);
  A.dbg_rays = dbg_rec ? dbg_rays : 0;
  A.dbg_cap = dbg_cap; A.dbg_counts = dbg_counts; A.dbg_rec = dbg_rec;
  launch_render<false>(A, grid, kSmemFwd, st);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_backward(const rg_gaussians& g, const rg_bvh& b, const rg_config& c,
                            const rg_rays* rays, const rg_camera* cam, const float* rgb,
                            const float* T, const int32_t* replay, const void* log,
                            size_t log_bytes, const float* d_rgb,
                            const rg_gaussian_grads& grads, rg_stats* stats, float* gbuf,
                            cudaStream_t st) {
  (void)T;
  RenderArgs A = {};
  A.S = view_of(b);
  A.c = c;
  dim3 grid;
  ray_grid(A, rays, cam, grid);
  set_log(A, log, log_bytes, A.n_rays);
  const int gs = grad_stride(b.sh_degree, b.sg_count);
  if (b.n > 0) cudaMemsetAsync(gbuf, 0, sizeof(float) * (size_t)gs * b.n, st);
  A.stats = stats;
  A.rgb_in = rgb; A.replay_in = replay; A.d_rgb = d_rgb; A.gbuf = gbuf; A.gstride = gs;
  if (A.n_rays > 0) { launch_render<true>(A, grid, kSmemBwd, st); count_launches(1); }
  if (b.n > 0) {
    k_finalize<<<(b.n + 255) / 256, 256, 0, st>>>(gbuf, gs, b.order, g, grads, stats);
    const int ablocks = (int)std::min<long long>(((long long)b.n + 7) / 8, 148 * 16);
    k_finalize_app<<<ablocks, 256, 0, st>>>(gbuf, gs, b.order, g, grads, stats);
    count_launches(2);
  }
  return cudaGetLastError();
}

cudaError_t launch_l1(const float* rgb, const float* target, int64_t n, float scale, float* d_rgb,
                      float* loss, cudaStream_t st) {
  if (n > 0) {
    const int64_t nb = (n + 255) / 256; const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
    k_l1<<<blocks, 256, 0, st>>>(rgb, target, n, scale, d_rgb, loss);
    count_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace rg

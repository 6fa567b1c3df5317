// Event-based generic tracker: block-local event queues (§2.3, re-designed
// for sm_100a).
//
// Shift's GPU transport runs every tracking operation as a kernel over a masked vector of
// histories.  Here one persistent block owns S particle slots (state in shared memory, SoA) and
// keeps them in per-event queues: reflected slots (no event), change_direction (absorption or
// isotropic scatter), find_cell / cross_surface descents (Alg. 7-8) at CSG levels, then
// at array levels, and free slots (births: pid claims with a warp-aggregated atomic on the global
// counter).  A warp takes up to 32 slots of ONE queue, so it runs one event type at a time, and
// then runs MOVE on the same slots: distance_to_boundary over all levels + collide-or-cross +
// move_within_cell + track-length tally (Table 1, Alg. 2).  Each slot is then appended
// to the queue of its next event with match.any / ballot / popc and one shared atomic per target.
//
// Two forms of the queues:
//  * ASYNC (the default, `NT_ROUNDS` unset): each queue is a ring in shared memory with a head and
//    a tail counter and no block barrier.  A warp reads the five heads, claims up to 32 entries of
//    the fullest ring (CAS on its head), and publishes every slot it appends to a lap-tagged ring
//    entry after a block fence (ring_publish / ring_take).  S may exceed the thread count (320 slots for 256 threads), so a
//    warp that finishes its chunk finds queued slots instead of waiting for other warps' chunks.
//  * rounds (`NT_ROUNDS`): one queue set per round sorted by event type, warps take consecutive
//    32-slot chunks, one block barrier per round, triple-buffered uint8 queues (S == B <= 256).
//
// The per-level universe stack of each slot stays in shared memory between stages; nothing
// round-trips through HBM.  Arithmetic is exactly the generic tracker's (nt_geom.cuh, descend(),
// level_distances()), so results are bit-identical to it and to the oracle.
#pragma once

NT_DEV_BEGIN

// Queue layout (uint8 slot indices), triple-buffered by round:
//   Q_M[p] move-ready, Q_C[p] collide, Q_DC[p] CSG descents, Q_DA[p] array descents, Q_F[p] free
enum { Q_M = 0, Q_C = 1, Q_DC = 2, Q_DA = 3, Q_F = 4, NQ = 5 };
// ASYNC with NR = 7 rings (models whose histories sit at different depths, e.g. a hex core inside a
// CSG reflector): collide and CSG-descent slots of histories above the deepest level go to rings
// of their own, so that a warp's MOVE runs slots with the same number of levels (the level loop
// otherwise diverges).  Ring q serves event kind ring_kind(q).
enum { Q_C2 = 5, Q_DC2 = 6 };
__host__ __device__ constexpr int ring_kind(int q) { return (0x0421045 >> (4 * q)) & 15; }   // 5 4 0 1 2 4 0
#ifndef NT_RING_SLEEP_NS
#define NT_RING_SLEEP_NS 64     // back-off of a warp that found every ring empty
#endif
using QIdx = uint8_t;           // rounds form: slot index in a queue (S == B <= 256 slots); the
                                // ASYNC rings hold slot + 1 in uint16 entries (S <= 512)

__device__ __forceinline__ int warp_append(bool pred, int* counter, int lane) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (m == 0) return -1;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return pred ? base + __popc(m & ((1u << lane) - 1u)) : -1;
}

__device__ __forceinline__ void warp_count(bool pred, unsigned int* counter, int lane) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (lane == 0 && m) atomicAdd(counter, (unsigned)__popc(m));
}

// ring capacity: the smallest power of two >= the slot count.  A slot is in at most one ring at a
// time, so at most S <= RB positions of a ring are allocated and unclaimed (tail - head <= S): when
// position p is allocated, position p - RB has already been claimed (see ring_publish / ring_take).  Positions are 32-bit
// counters; 2^32 is a multiple of 128 RB, so lap tags stay consistent across the wrap.
__host__ __device__ constexpr int ring_size(int S) { return S <= 128 ? 128 : S <= 256 ? 256 : 512; }

// Frames T_l of the universe stack: stored per slot (3 doubles per level >= 1), or recomputed from
// the stack's cells / tiles with the descent's own arithmetic (NT_FRAMES_RECOMPUTE: 72 B less per
// slot at depth 4, so that four 256-thread blocks fit an SM).  Bit-identical either way.
#ifndef NT_FRAMES_RECOMPUTE
#define NT_FRAMES_RECOMPUTE (NT_FEAT != 0)   // f7 (hex / plane / sphere models): recomputed, for more slots
#endif
constexpr bool kFramesRecompute = NT_FRAMES_RECOMPUTE != 0;
// Frames stored only below arrays; below a CSG level recomputed from the parent's frame and cell
// translation (one uniform-ish load per axis instead of a bank-conflicted shared load).
#ifndef NT_FRAMES_MIXED
#define NT_FRAMES_MIXED 0
#endif
// EVENT -> MOVE forwarding: the position a descent or birth just read or made, the flags / depth /
// material cell a descent produced, and the direction and tau a birth or scatter drew stay in
// registers for the MOVE of the same slot instead of a shared-memory store and reload (bank
// conflicts on every per-slot access: profiles/r02_ncu_analysis.md).  0: always reload.
#ifndef NT_FORWARD
#define NT_FORWARD 1
#endif
constexpr bool kForward = NT_FORWARD != 0;
#ifndef NT_DEPTH_RINGS
#define NT_DEPTH_RINGS 1     // depth-class rings (NR = 7) for the f7 feature set (0: five rings everywhere)
#endif
// depth-class rings for the f0 feature set as well (with the safety skip, a chunk that mixes depths
// runs the shallow lanes' upper levels beside the deep lanes' lower ones)
#ifndef NT_DEPTH_RINGS_F0
#define NT_DEPTH_RINGS_F0 0
#endif
// Safety skip of the upper levels: MOVE evaluates levels [lk, L) with lk = L - 2 and
// skips levels [0, lk) when the slot's stored safety bound proves that none of their candidates can
// win, tie or near-tie; otherwise the slot is deferred with its partial winner to the U ring, whose
// chunks evaluate the upper levels, merge, and refresh the bound.  Bit-identical to evaluating all
// levels.  0: every MOVE evaluates every level.
#ifndef NT_SAFETY
#define NT_SAFETY 0          // measured slower on every config (profiles/r02_experiments.md rows 54-57)
#endif
constexpr bool kSafeSP = NT_SAFETY != 0 && !kFramesRecompute && NT_FRAMES_MIXED == 0;   // SP ring kernels
// slots per block of the big-slot ring variant: 320 with stored frames (288 with the safety skip's 12
// extra bytes per slot and its ring), 384 with recomputed frames (147 B per slot at depth 4), so that
// three 256-thread blocks still fit an SM at depth <= 4
#ifndef NT_SLOTS_BIG
#define NT_SLOTS_BIG (kFramesRecompute ? 384 : kSafeSP ? 288 : 320)
#endif
constexpr int kSlotsBig = NT_SLOTS_BIG;
// threads per block of the big-slot SP ring kernel without trace (tuning: fewer warps per block
// leave more queued slots per warp)
#ifndef NT_RING_THREADS
#define NT_RING_THREADS 256
#endif
constexpr int kRingThreads = NT_RING_THREADS;
// deep models whose 320-slot blocks do not fit three to an SM (f0, depth 5): two blocks of 320 threads
// with 400 slots each (the same 20 warps' worth of queued slots per warp as 320 / 256) instead of 256 slots
constexpr int kDeepThreads = 320, kDeepSlots = 400;
// queues one chunk may draw from (1: the fullest only; 2: topped up from the next fullest)
#ifndef NT_CLAIM_RINGS
#define NT_CLAIM_RINGS 1     // 2 measured slower on C2 / C3 / C5r (profiles/r02_experiments.md row 62)
#endif
// a chunk smaller than NT_CLAIM_MIN waits (back-off) up to NT_CLAIM_WAIT times for its queue to fill
#ifndef NT_CLAIM_MIN
#define NT_CLAIM_MIN 0
#endif
#ifndef NT_CLAIM_WAIT
#define NT_CLAIM_WAIT 0
#endif
constexpr int kClaimRings = NT_CLAIM_RINGS;
// levels the safety skip covers at most: lk = min(NT_SAFE_K, L - 2) (the two deepest levels are
// always evaluated)
#ifndef NT_SAFE_K
#define NT_SAFE_K 2
#endif
constexpr int kQN = 18;              // ints for ring heads / tails (2 * rings <= 16) or rounds queue counts (3 NQ)
constexpr double kSafeRel = 1e-6;    // skip only if safety * (1 - kSafeRel) > d_lower + kSafeAbs
constexpr double kSafeAbs = 1e-9;    // (cm) > kFlagDist: the F2 near-tie window stays exact

size_t event_smem_bytes(const DevGeom& g, int B, bool trace, bool async = false, bool store_t = true, int nr = NQ,
                        bool safety = false) {
  const size_t nmc = g.n_mc, d = g.max_depth;
  size_t s = 0;
  s += (7 + (store_t ? 3 * (d - 1) : 0) + (trace ? 1 : 0) + (safety ? 1 : 0)) * 8 * (size_t)B;   // doubles (T from level 1)
  s += (6 + 4 * d + (trace ? 2 : 0) + (safety ? 1 : 0)) * 4 * (size_t)B;   // ints
  s += (3 + (trace ? 1 : 0)) * (size_t)B;                             // bytes
  s = (s + 15) & ~size_t(15);
  if (async) s += (nr + (safety ? 1 : 0)) * sizeof(uint16_t) * (size_t)ring_size(B);   // ring queues
  else s += 3 * NQ * sizeof(QIdx) * (size_t)B;                        // queues (triple-buffered)
  s += (nmc + kNC + kQN + 4) * 4;                                       // exits, counters, queue counts
  return (s + 15) & ~size_t(15);
}

__device__ __forceinline__ uint32_t vload(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ uint32_t vload(const uint16_t* p) { return *reinterpret_cast<const volatile uint16_t*>(p); }
__device__ __forceinline__ void vstore(uint16_t* p, uint32_t v) {
  *reinterpret_cast<volatile uint16_t*>(p) = static_cast<uint16_t>(v);
}
// Ring entries (ASYNC form) carry a lap tag, so that producers and consumers of different laps of
// the same entry can never act on each other's state (a sequence-numbered MPMC ring with plain
// 16-bit loads and stores, no atomics on the entries).  Position p of a ring maps to entry
// p mod RB and belongs to lap L = p / RB; tag(L) = L mod 128.  An entry is
//   FREE(L) = tag(L) << 9 | 511   : empty, next to be filled by the producer of lap L;
//   FULL(L) = tag(L) << 9 | slot  : holds the slot pushed at lap L (slot <= 510).
// The producer of position p waits for FREE(L) and stores FULL(L); the consumer of p waits for
// FULL(L) and stores FREE(L + 1).  So each value is put by the one producer of its position and
// taken by the one consumer of its position, in lap order.  Tags alias only if two parties of the
// same entry were 128 laps apart.  They cannot be: at any moment the positions of one entry that
// are in progress (allocated but not yet consumed) are the at most one allocated-unclaimed position
// (tail - head <= S <= RB) plus one per warp (a warp takes and pushes consecutive positions of a ring,
// so it holds at most one position per entry), i.e. at most warps + 1 < 128 laps apart.
// Progress: the lap-L producer of an entry waits only for the lap-(L-1) consumer, which has claimed
// its position (see above) and waits only for the lap-(L-1) producer: by induction the oldest
// in-progress position of every entry can always advance.  (tail - head <= S <= RB, so when p is
// allocated the head is past p - RB.)
// stored safety word: a float at or below the bound with the covered level count in its three low
// mantissa bits.  v (1 - 2^-40) rounded down to float stays below the exact v despite the rounding of
// the running subtraction that produced v; clearing the low bits and stepping 8 ulp down keeps the
// value with the count OR-ed in below it.  0 = no bound.
__device__ __forceinline__ uint32_t ss_pack(double v, int cov) {
  const float f = __double2float_rd(v * (1.0 - 0x1p-40));
  const uint32_t m = f > 1e-30f ? (__float_as_uint(f) & ~7u) - 8u : 0u;
  return m | static_cast<uint32_t>(cov);
}

constexpr uint32_t kRingFree = 511u;
__device__ __forceinline__ uint32_t ring_tag(uint32_t pos, int log2rb) { return ((pos >> log2rb) & 127u) << 9; }
__device__ __forceinline__ void ring_publish(uint16_t* e, uint32_t pos, int log2rb, int slot) {
  const uint32_t tag = ring_tag(pos, log2rb);
  while (vload(e) != (tag | kRingFree)) {}
  vstore(e, tag | static_cast<uint32_t>(slot));
}
__device__ __forceinline__ int ring_take(uint16_t* e, uint32_t pos, int log2rb) {
  const uint32_t tag = ring_tag(pos, log2rb);
  uint32_t v;
  while (((v = vload(e)) & ~kRingFree) != tag || (v & kRingFree) == kRingFree) {}
  vstore(e, ring_tag(pos + (1u << log2rb), log2rb) | kRingFree);
  return static_cast<int>(v & kRingFree);
}

// DP = true: the tracking operations go through the virtual tracker objects (dp_tracker.cuh).
// TALLY: bit 0 mesh tally (M1), bit 1 per-instance tally (D1); separate instantiations.
// ASYNC = true: no rounds and no block barrier.  Each queue is a ring of B entries with a head
// and a tail counter in shared memory; a warp claims up to 32 entries of the fullest queue (CAS on
// the head), runs that EVENT and MOVE on them, and appends every slot to the ring of its next
// event (warp-aggregated atomic on the tail, entry published after a block fence).  The block
// ends when the pids are exhausted and no history is live.
// S = particle slots per block (ASYNC only: S may exceed B, so that a warp finishing its chunk finds
// other slots queued instead of waiting for the chunks other warps hold; rounds need S == B).
// RTK = 0: generic tracker; 1 / 2: the rect-specialised tracker (rect_geom.cuh, Alg. 9-10) with a box /
// CZ-annuli root, run by the same scheduler (rg describes the model; unused when RTK = 0).
#ifndef NT_EVENT_MINB
#define NT_EVENT_MINB 3     // blocks per SM the 256-thread kernels are compiled for (tuning builds)
#endif
template <int B, bool TRACE, bool STATES, bool DP = false, int TALLY = 0, bool ASYNC = false, int S = B, int RTK = 0,
          int NR = NQ>
__global__ void __launch_bounds__(B, B == kDeepThreads && S == kDeepSlots ? 2 : B >= 256 || S > B ? NT_EVENT_MINB : 5)
k_track_event(const DevGeom g, const KRun R, const RectGeom rg) {
  static_assert(ASYNC || S == B, "round-based queues need one slot per thread");
  static_assert(RTK == 0 || (!DP && !(TALLY & 2)), "RTK: SP dispatch, no instance tallies");
  static_assert(NR == NQ || (ASYNC && NR == 7), "depth-class rings: ring scheduler only, 7 rings");
  static_assert(ring_kind(Q_C2) == 4 && ring_kind(Q_DC2) == 0 && ring_kind(Q_F) == 2 && Q_DC2 < 7, "ring table");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nmc = g.n_mc, maxd = g.max_depth;
  constexpr bool kStoreT = RTK != 0 || DP || !kFramesRecompute;   // frames in shared memory
  constexpr bool kMixedT = kStoreT && RTK == 0 && !DP && NT_FRAMES_MIXED != 0;
  // safety skip of the upper levels: generic SP tracker on the ring scheduler with stored frames
  constexpr bool kSafe = kSafeSP && ASYNC && !DP && RTK == 0 && kStoreT && !kMixedT;
  constexpr int NRT = NR + (kSafe ? 1 : 0);     // rings, the U ring (deferred upper levels) last
  constexpr int QU = NR;
  static_assert(2 * NRT <= kQN, "ring heads and tails");
  // ---- carve shared memory (see event_smem_bytes)
  double* sx = reinterpret_cast<double*>(smem);
  double* sy = sx + S; double* sz = sy + S; double* su = sz + S; double* sv = su + S; double* sw = sv + S;
  double* stau = sw + S;
  double* sTb = stau + S;                           // [maxd-1][3][S] (T_0 = 0)
  double* sps = sTb + (kStoreT ? 3 * (maxd - 1) * S : 0);   // TRACE: pending segment length
  double* sdl = sps + (TRACE ? S : 0);              // kSafe: deferred slot's lower-level winner distance
  uint32_t* sidx = reinterpret_cast<uint32_t*>(sdl + (kSafe ? S : 0));
  uint32_t* sepoch = sidx + S; uint32_t* snseg = sepoch + S;
  int32_t* smc = reinterpret_cast<int32_t*>(snseg + S);
  int32_t* sos = smc + S;                           // on-surface sid (-1 none)
  int32_t* sdesc = sos + S;                         // pending descent: l0 | fsense<<4 | (fh+1)<<5 (CSG: half-space, array: face)
  int32_t* sib = sdesc + S;                         // [maxd][4][S]
  int32_t* spj = sib + 4 * maxd * S;                // TRACE: pending j, cell_before
  int32_t* spcb = spj + (TRACE ? S : 0);
  uint32_t* sss = reinterpret_cast<uint32_t*>(spcb + (TRACE ? S : 0));   // kSafe: safety word (see ss_pack)
  uint8_t* sflags = reinterpret_cast<uint8_t*>(sss + (kSafe ? S : 0));
  uint8_t* sL = sflags + S;
  int8_t* sosl = reinterpret_cast<int8_t*>(sL + S);
  int8_t* spl = sosl + S;                           // TRACE: pending level
  size_t off = (size_t)(reinterpret_cast<unsigned char*>(spl + (TRACE ? S : 0)) - smem);
  off = (off + 15) & ~size_t(15);
  QIdx* sq = reinterpret_cast<QIdx*>(smem + off);            // [3][NQ][S]        (rounds)
  constexpr int RB = ring_size(S);
  constexpr int kLog2RB = RB == 128 ? 7 : RB == 256 ? 8 : 9;
  static_assert(S <= 510 && (1 << kLog2RB) == RB, "ring entries hold slot <= 510");
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem + off);  // [NRT][RB] lap-tagged entries (ASYNC)
  unsigned int* s_exit = ASYNC ? reinterpret_cast<unsigned int*>(ring + NRT * RB)
                               : reinterpret_cast<unsigned int*>(sq + 3 * NQ * S);
  unsigned int* s_cnt = s_exit + nmc;
  int* s_qn = reinterpret_cast<int*>(s_cnt + kNC);          // [3][NQ] (rounds)
  int* s_flag = s_qn + kQN;                                 // [0] = pids exhausted, [1] live (ASYNC)
  uint32_t* a_head = reinterpret_cast<uint32_t*>(s_qn);      // ASYNC: [NRT] heads, [NRT] tails (2 NRT <= kQN)
  uint32_t* a_tail = a_head + NRT;
  double* gl = R.slices + (size_t)blockIdx.x * nmc;         // per-block track-length tally (global)

  for (int i = tid; i < nmc; i += B) s_exit[i] = 0u;
  for (int i = tid; i < kNC; i += B) s_cnt[i] = 0u;
  if (tid < kQN) s_qn[tid] = (!ASYNC && tid == 0 * NQ + Q_F) ? B : 0;   // rounds: round 0 reads set 0, all free
  if (ASYNC) {
    for (int i = tid; i < NRT * RB; i += B) ring[i] = static_cast<uint16_t>(kRingFree);     // FREE(lap 0)
    __syncthreads();
    for (int i = tid; i < S; i += B) ring[Q_F * RB + i] = static_cast<uint16_t>(i);        // FULL(lap 0): all slots free
    if (tid == 0) { a_tail[Q_F] = S; s_flag[0] = 0; s_flag[1] = 0; }
  } else {
    if (tid == 0) s_flag[0] = 0;
    for (int i = tid; i < B; i += B) sq[(0 * NQ + Q_F) * B + i] = static_cast<QIdx>(i);   // round 0 reads set 0: all slots free
  }
  __syncthreads();

  auto Q = [&](int p, int q) { return sq + (p * NQ + q) * B; };
  auto QN = [&](int p, int q) -> int& { return s_qn[p * NQ + q]; };
  const uint32_t max_seg = static_cast<uint32_t>(R.max_seg);

  // history ended: per-history counters and per-particle outputs (slot becomes free)
  auto finalize = [&](int slot, int term) {
    atomicAdd(s_cnt + C_PART, 1u);
    atomicAdd(s_cnt + (term == NT_T_ABSORBED ? C_ABS : term == NT_T_LEAKED ? C_LEAK : term == NT_T_LOST ? C_LOST : C_CAP), 1u);
    const uint32_t fl = sflags[slot];
    if (fl) atomicAdd(s_cnt + C_FLAG, 1u);
    const uint32_t id = sidx[slot];
    if (R.pflags) R.pflags[id] = static_cast<uint8_t>(fl);
    if (R.pnseg) R.pnseg[id] = snseg[slot];
    if (R.pterm) R.pterm[id] = static_cast<uint8_t>(term);
    atomicAdd(s_cnt + C_SEG, snseg[slot]);
    if (ASYNC) atomicSub(reinterpret_cast<unsigned int*>(s_flag + 1), 1u);   // one history fewer live
  };

  for (int round = 0;; ++round) {
    // queues triple-buffered by round: read rd (filled in round-1), append wr, reset rs
    const int rd = round % 3, wr = (round + 1) % 3, rs = (round + 2) % 3;
    int nmv = 0, nco = 0, ndc = 0, nda = 0, nfr = 0, total = 32;
    if (!ASYNC) {
      if (tid == 0)
        for (int k = 0; k < NQ; ++k) QN(rs, k) = 0;          // read in round-1, refilled in round+1
      nmv = QN(rd, Q_M); nco = QN(rd, Q_C); ndc = QN(rd, Q_DC); nda = QN(rd, Q_DA); nfr = QN(rd, Q_F);
      total = nmv + nco + ndc + nda + nfr;
    }
    for (int base = ASYNC ? 0 : warp * 32; base < total; base += B) {
      const int i = base + lane;
      // kind: 5 move only (reflected), 4 collide, 0 CSG descent, 1 array descent, 2 birth, 3 none,
      // 6 deferred MOVE (kSafe: upper levels + merge)
      int slot = 0, kind = 3;
      bool valid = i < total;
      if constexpr (ASYNC) {
        // ---- claim up to 32 entries of the fullest queue (lane 0), or finish
        // lane k < NQ reads queue k; the fullest queue (lowest index on ties) wins a warp max-reduction.
        // Top-up (kClaimRings > 1): a chunk short of 32 takes the rest from the next fullest queue(s);
        // lanes then run different EVENT kinds (each kind's code runs once, as in separate chunks),
        // but one MOVE serves all of them.
        int q = -1, q2 = -1;
        uint32_t h = 0, take = 0, h2 = 0, take2 = 0;
        int waits = 0;
        for (;;) {
          const bool births = vload(reinterpret_cast<uint32_t*>(s_flag)) == 0u;
          uint32_t hk = 0, av = 0;
          if (lane < NRT && (lane != Q_F || births)) { hk = vload(a_head + lane); av = vload(a_tail + lane) - hk; }
          const uint32_t mx = __reduce_max_sync(0xffffffffu, (av << 8) | static_cast<uint32_t>(255 - lane));
          const uint32_t bav = mx >> 8;                  // av <= S slots (< 2^24): fits above the lane byte
          if (NT_CLAIM_MIN > 0 && bav > 0u && bav < NT_CLAIM_MIN && waits < NT_CLAIM_WAIT) {
            ++waits;
            __nanosleep(NT_RING_SLEEP_NS);
            continue;
          }
          if (bav > 0u) {
            const int best = 255 - static_cast<int>(mx & 255u);
            const uint32_t bh = __shfl_sync(0xffffffffu, hk, best);
            const uint32_t tk = bav < 32u ? bav : 32u;
            int won = 0;
            if (lane == 0) won = atomicCAS(a_head + best, bh, bh + tk) == bh;
            if (__shfl_sync(0xffffffffu, won, 0)) {
              q = best; h = bh; take = tk;
              if (kClaimRings > 1 && tk < 32u) {
                // second fullest queue (availability as read above; the head CAS validates it)
                const uint32_t a2 = lane == best ? 0u : av;
                const uint32_t mx2 = __reduce_max_sync(0xffffffffu, (a2 << 8) | static_cast<uint32_t>(255 - lane));
                if ((mx2 >> 8) > 0u) {
                  const int b2 = 255 - static_cast<int>(mx2 & 255u);
                  const uint32_t hb2 = __shfl_sync(0xffffffffu, hk, b2);
                  const uint32_t want = 32u - tk, tk2 = (mx2 >> 8) < want ? (mx2 >> 8) : want;
                  int won2 = 0;
                  if (lane == 0) won2 = atomicCAS(a_head + b2, hb2, hb2 + tk2) == hb2;
                  if (__shfl_sync(0xffffffffu, won2, 0)) { q2 = b2; h2 = hb2; take2 = tk2; }
                }
              }
              break;
            }
            continue;
          }
          if (!births && vload(reinterpret_cast<uint32_t*>(s_flag + 1)) == 0u) break;   // all done
          __nanosleep(NT_RING_SLEEP_NS);
        }
        if (q < 0) break;
        valid = static_cast<uint32_t>(lane) < take + take2;
        if (valid) {
          const bool second = static_cast<uint32_t>(lane) >= take;
          const int ql = second ? q2 : q;
          const uint32_t pos = second ? h2 + (lane - take) : h + lane;
          slot = ring_take(ring + ql * RB + (pos & (RB - 1)), pos, kLog2RB);
          kind = kSafe && ql == QU ? 6 : ring_kind(ql);   // Q_M, Q_C, Q_DC, Q_DA, Q_F (, Q_C2, Q_DC2) (, Q_U) -> 5 4 0 1 2 (4 0) (6)
        }
        __threadfence_block();
      } else if (valid) {
        if (i < nmv) { slot = Q(rd, Q_M)[i]; kind = 5; }
        else if (i < nmv + nco) { slot = Q(rd, Q_C)[i - nmv]; kind = 4; }
        else if (i < nmv + nco + ndc) { slot = Q(rd, Q_DC)[i - nmv - nco]; kind = 0; }
        else if (i < nmv + nco + ndc + nda) { slot = Q(rd, Q_DA)[i - nmv - nco - ndc]; kind = 1; }
        else { slot = Q(rd, Q_F)[i - nmv - nco - ndc - nda]; kind = 2; }
      }
      // append this lane's slot to queue q of the next event (warp-aggregated)
      auto push = [&](int qq, bool pred) {
        if constexpr (ASYNC) {
          const unsigned m = __ballot_sync(0xffffffffu, pred);
          if (m) {
            const int leader = __ffs(m) - 1;
            uint32_t base2 = 0;
            if (lane == leader) base2 = atomicAdd(a_tail + qq, static_cast<uint32_t>(__popc(m)));
            base2 = __shfl_sync(0xffffffffu, base2, leader);
            if (pred) {
              __threadfence_block();                               // slot state before the entry
              const uint32_t pos = base2 + __popc(m & ((1u << lane) - 1u));
              ring_publish(ring + qq * RB + (pos & (RB - 1)), pos, kLog2RB, slot);
            }
          }
        } else {
          const int pos = warp_append(pred, &QN(wr, qq), lane);
          if (pos >= 0) Q(wr, qq)[pos] = static_cast<QIdx>(slot);
        }
      };
      // ASYNC: append every lane's slot to its target ring in one pass (lanes grouped by target
      // with match.any; one tail atomic per target; -1 = no target)
      auto push_all = [&](int qq) {
        if (!__any_sync(0xffffffffu, qq >= 0)) return;
        const unsigned grp = __match_any_sync(0xffffffffu, qq);
        const int leader = __ffs(grp) - 1;
        uint32_t base2 = 0;
        if (qq >= 0 && lane == leader) base2 = atomicAdd(a_tail + qq, static_cast<uint32_t>(__popc(grp)));
        base2 = __shfl_sync(0xffffffffu, base2, leader);
        if (qq >= 0) {
          __threadfence_block();                                   // slot state before the entry
          const uint32_t pos = base2 + __popc(grp & ((1u << lane) - 1u));
          ring_publish(ring + qq * RB + (pos & (RB - 1)), pos, kLog2RB, slot);
        }
      };
      // ---------------- EVENT: change_direction / descent / birth of this chunk's slots
        // births: claim pids for this warp's birth lanes (warp-aggregated)
        const unsigned bm = __ballot_sync(0xffffffffu, kind == 2);
        bool born = false;
        if (bm) {
          const int leader = __ffs(bm) - 1;
          unsigned long long b0 = 0;
          if (lane == leader) b0 = atomicAdd(R.counter, static_cast<unsigned long long>(__popc(bm)));
          b0 = __shfl_sync(0xffffffffu, b0, leader);
          if (kind == 2) {
            const unsigned long long id = b0 + __popc(bm & ((1u << lane) - 1u));
            if (id < R.n) { born = true; sidx[slot] = static_cast<uint32_t>(id); }
            else s_flag[0] = 1;                          // pids exhausted: slot stays unused
          }
          if (ASYNC) {
            const unsigned nb = __ballot_sync(0xffffffffu, born);
            if (lane == leader && nb) atomicAdd(reinterpret_cast<unsigned int*>(s_flag + 1), static_cast<unsigned>(__popc(nb)));
          }
        }
        bool ok = false, done = false, scat = false, absorbed = false;
        int iso_ep = -2;      // >= 0: isotropic direction from (epoch iso_ep, block 1) and tau; -1: tau only
        double xtau = 0.0;
        // forwarded to MOVE (kForward): position, direction, tau, and a descent's flags / depth / cell
        double fx = 0.0, fy = 0.0, fz = 0.0, fu = 0.0, fv = 0.0, fw = 0.0, ftau = 0.0;
        uint32_t fflags = 0;
        int fL = 0, fmc = 0;
        bool f_pos = false, f_dir = false, f_tau = false, f_desc = false;
        if (kind == 4) {
          // ---- change_direction (O14, O15)
          const uint64_t pid = R.pid0 + sidx[slot];
          const uint32_t epoch = sepoch[slot] + 1;
          sepoch[slot] = epoch;
          const int mc = smc[slot];
          double xa, xb;
          draw2(R.seed, pid, epoch, 0, xa, xb);
          const int cb = TRACE ? ld(g.mc_cell + mc) : 0;
          if (xa < ld(g.mc_pabs + mc)) {
            absorbed = true;
            if (R.bank) bank_sites(g, R.bank, R.bank_n, mc, sidx[slot], xb, sx[slot], sy[slot], sz[slot]);
            if (TRACE) emit<TRACE>(R, pid, snseg[slot] - 1, NT_EV_COLLIDE, -1, -1, cb, cb, sps[slot], NT_T_ABSORBED, sflags[slot]);
            finalize(slot, NT_T_ABSORBED);
          } else {
            iso_ep = static_cast<int>(epoch);      // direction and tau: shared tail below
            xtau = xb;
            scat = true;
            if (TRACE) emit<TRACE>(R, pid, snseg[slot] - 1, NT_EV_COLLIDE, -1, -1, cb, cb, sps[slot], NT_T_NONE, sflags[slot]);
          }
        } else if (kind == 0 || kind == 1 || born) {
          Stack st;
          st.si = sib + slot;
          st.sT = sTb + slot;
          st.B = S;
          double rx = 0, ry = 0, rz = 0;
          uint32_t flags = 0;
          int L = 0, mc = 0;
          int l0 = 0, du = g.root, fh = -1, fsense = 0;
          double Tx = 0.0, Ty = 0.0, Tz = 0.0;
          if (born) {
            const uint64_t pid = R.pid0 + sidx[slot];
            double xa;
            draw2(R.seed, pid, 0, 0, xa, xtau);
            if (STATES) {
              const uint64_t id = sidx[slot];
              rx = R.states[id]; ry = R.states[R.n + id]; rz = R.states[2 * R.n + id];
              fu = R.states[3 * R.n + id]; fv = R.states[4 * R.n + id]; fw = R.states[5 * R.n + id];
              su[slot] = fu; sv[slot] = fv; sw[slot] = fw;
              f_dir = kForward;
              iso_ep = -1;                         // tau only
            } else {
              double xx, xy, xz, unused;
              draw2(R.seed, pid, 0, 2, xx, xy);
              draw2(R.seed, pid, 0, 3, xz, unused);
              rx = R.lo[0] + R.w[0] * xx;
              ry = R.lo[1] + R.w[1] * xy;
              rz = R.lo[2] + R.w[2] * xz;
              iso_ep = 0;                          // epoch-0 direction (block 1) in the shared tail
            }
            if (!kForward) { sx[slot] = rx; sy[slot] = ry; sz[slot] = rz; }   // else MOVE stores it
            sepoch[slot] = 0; snseg[slot] = 0; sos[slot] = -1; sosl[slot] = -1;
            if (TRACE) spl[slot] = -2;
          } else {
            rx = sx[slot]; ry = sy[slot]; rz = sz[slot];
            flags = sflags[slot];
            const int dsc = sdesc[slot];
            l0 = dsc & 15;
            fsense = (dsc >> 4) & 1;
            fh = (dsc >> 5) - 1;
            if constexpr (kMixedT) {
              frame_mixed(g, st, l0, Tx, Ty, Tz);
            } else if constexpr (kStoreT) {
              Tx = st.T(l0, 0); Ty = st.T(l0, 1); Tz = st.T(l0, 2);
            } else {
              frame_of(g, st, l0, Tx, Ty, Tz);
            }
            if (kind == 0) {
              du = st.u(l0);
            } else {                                     // Alg. 6: tile +- 1 at level l0, then daughter
              const int j = fh;
              int ta = st.a(l0), tb = st.b(l0), tc = st.c(l0);
              double tx, ty, tz;
              if constexpr (DP) {
                du = get_tracker(g, st.u(l0))->next_tile(g, j, ta, tb, tc, tx, ty, tz);
              } else {
                const DUniv* U = g.univ + st.u(l0);
                const int uk = st.ukind(l0);
                if (!kHex || uk == U_RECT) {
                  const int dir = (j & 1) ? 1 : -1, ax = j >> 1;
                  if (ax == 0) ta += dir; else if (ax == 1) tb += dir; else tc += dir;
                } else if (j < 6) {
                  ta += (j == 0 || j == 5) ? 1 : ((j == 2 || j == 3) ? -1 : 0);
                  tb += (j == 1 || j == 2) ? 1 : ((j == 4 || j == 5) ? -1 : 0);
                } else {
                  tc += (j == 7) ? 1 : -1;
                }
                du = array_daughter(g, U, uk, ta, tb, tc, tx, ty, tz);
              }
              st.a(l0) = ta; st.b(l0) = tb; st.c(l0) = tc;
              Tx = Tx + tx; Ty = Ty + ty; Tz = Tz + tz;
              l0 = l0 + 1;
              fh = -1;
              fsense = 0;
            }
          }
          if constexpr (DP) ok = du >= 0 && descend_dp(g, st, l0, du, Tx, Ty, Tz, rx, ry, rz, fh >= 0 ? hs_sid(ld(&g.hsr[fh].e)) : -1,
                                                       fsense, L, mc, flags);
          else if constexpr (RTK != 0) {
            // RTK: a CSG crossing's key is the surface id itself; an array step stores the new
            // tile's daughter and frame, then the unrolled descent continues below it
            if (kind == 1 && du >= 0) {
              st.set_u(l0, du, l0 <= rg.K ? U_RECT : U_CSG);
              st.setT(l0, 0, Tx); st.setT(l0, 1, Ty); st.setT(l0, 2, Tz);
            }
            ok = du >= 0 && rect_descend<RTK == 1>(g, rg, st, l0, fh, fsense, rx, ry, rz, L, mc, flags);
          }
          else ok = du >= 0 && descend<kStoreT, kMixedT>(g, st, l0, du, Tx, Ty, Tz, rx, ry, rz, fh, fsense, L, mc, flags);
          done = true;
          if (!ok) flags |= NT_F3;
          if (!kForward || !ok) sflags[slot] = static_cast<uint8_t>(flags);   // ok + kForward: MOVE stores it
          if (ok) { sL[slot] = static_cast<uint8_t>(L); smc[slot] = mc; }
          if (kForward) {
            fx = rx; fy = ry; fz = rz; f_pos = true;
            fflags = flags; fL = L; fmc = mc; f_desc = ok;
          }
          if (TRACE) {
            const uint64_t pid = R.pid0 + sidx[slot];
            const int pl = spl[slot];
            if (pl == -2) {
              if (!ok) emit<TRACE>(R, pid, 0, NT_EV_CROSS, -1, -1, -1, -1, 0.0, NT_T_LOST, flags);
            } else {
              emit<TRACE>(R, pid, snseg[slot] - 1, NT_EV_CROSS, pl, spj[slot], spcb[slot],
                          ok ? ld(g.mc_cell + mc) : -1, sps[slot], ok ? NT_T_NONE : NT_T_LOST, flags);
            }
          }
          if (!ok) finalize(slot, NT_T_LOST);
        }
      // one direction / tau site for births and scatters (O15, O12): keeps the kernel's code small
      if (iso_ep > -2) {
        if (iso_ep >= 0) {
          double xmu, xphi, u, v, w;
          draw2(R.seed, R.pid0 + sidx[slot], static_cast<uint32_t>(iso_ep), 1, xmu, xphi);
          isotropic(xmu, xphi, u, v, w);
          su[slot] = u; sv[slot] = v; sw[slot] = w;
          if (kForward) { fu = u; fv = v; fw = w; f_dir = true; }
        }
        if (kForward) { ftau = -spec_log(xtau); f_tau = true; }   // MOVE stores it (the slot moves, or ends)
        else stau[slot] = -spec_log(xtau);
      }
      const bool ready = kind == 5 || kind == 6 || (done && ok) || scat;
      const bool ended_at_event = (done && !ok) || absorbed;
      if (!ASYNC) push(Q_F, ended_at_event);
      // ---------------- MOVE the same slots (no barrier between a slot's event and its move)
      {
        // outcome: 0 none, 1 reflect (-> M), 2 collide, 3 CSG descent, 4 array descent, 5 ended,
        // 6 deferred to the U ring (kSafe: upper levels still to evaluate)
        int outc = 0, term = NT_T_NONE, lcross = -1;
        bool seg = false;
        if (ready) {
          Stack st;
          st.si = sib + slot;
          st.sT = sTb + slot;
          st.B = S;
          double rx, ry, rz, u, v, w, tau;
          uint32_t flags;
          int L, mc;
          if (f_pos) { rx = fx; ry = fy; rz = fz; } else { rx = sx[slot]; ry = sy[slot]; rz = sz[slot]; }
          if (f_dir) { u = fu; v = fv; w = fw; } else { u = su[slot]; v = sv[slot]; w = sw[slot]; }
          tau = f_tau ? ftau : stau[slot];
          if (f_desc) { flags = fflags; L = fL; mc = fmc; }
          else { flags = sflags[slot]; L = sL[slot]; mc = smc[slot]; }
          uint32_t nseg = snseg[slot];
          int os_l = sosl[slot], os_s = sos[slot];
          if (nseg >= max_seg) {
            flags |= NT_F3;
            term = NT_T_CAPPED;
            outc = 5;
            emit<TRACE>(R, R.pid0 + sidx[slot], nseg, NT_EV_COLLIDE, -1, -1, ld(g.mc_cell + mc), -1, 0.0,
                        NT_T_CAPPED, flags);
          } else {
            Best b;
            b.init();
            // kSafe modes: 0 LOWER (levels [lk, L), then skip or defer), 1 UPPER (U ring: levels [0, lk)
            // merged with the deferred lower winner), 2 FULL (births: every level)
            const int mode = !kSafe ? 2 : kind == 6 ? 1 : kind == 2 ? 2 : 0;
            const int lk = kSafe && L >= 3 ? min(NT_SAFE_K, L - 2) : 0;   // upper levels [0, lk)
            double lb = NT_INF;                                 // safety bound of [0, lk) (modes 1, 2)
            uint32_t ssw = 0;                                   // stored safety word (mode 0)
            bool near2 = false, defer = false;                  // O16 F2 runner-up test; mode 0 deferral
            if constexpr (RTK != 0) {
              rect_distances<RTK == 1>(g, rg, st, L, rx, ry, rz, u, v, w, os_l, os_s, b);
            } else {
              if constexpr (DP) {
                for (int l = 0; l < L; ++l) level_distances_dp(g, st, l, rx, ry, rz, u, v, w, os_l, os_s, b);
              } else if constexpr (kMixedT) {
                // stored frames below arrays, parent frame + cell translation below CSG levels
                double Tx = 0.0, Ty = 0.0, Tz = 0.0;
                int pkind = U_RECT, pcell = 0;
                for (int l = 0; l < L; ++l) {
                  if (l > 0) {
                    if (pkind == U_CSG) {
                      Tx = Tx + ld(g.cell_tr + 3 * pcell); Ty = Ty + ld(g.cell_tr + 3 * pcell + 1);
                      Tz = Tz + ld(g.cell_tr + 3 * pcell + 2);
                    } else {
                      Tx = st.T(l, 0); Ty = st.T(l, 1); Tz = st.T(l, 2);
                    }
                  }
                  const DUniv* U = g.univ + st.u(l);
                  const int kind_l = st.ukind(l), ia = st.a(l), ib = st.b(l), ic = st.c(l);
                  level_candidates(g, U, kind_l, ia, ib, ic, l, rx - Tx, ry - Ty, rz - Tz, u, v, w, os_l, os_s, b);
                  pkind = kind_l;
                  pcell = ia;
                }
              } else if constexpr (kSafe) {
                // the main loop is the plain one over [la, lz); the upper levels' safety bound is a
                // separate pass, run only by U-ring chunks and births (keeps the loop's registers)
                for (int l = mode == 0 ? lk : 0; l < (mode == 1 ? lk : L); ++l)
                  level_distances(g, st, l, rx, ry, rz, u, v, w, os_l, os_s, b);
                if (mode != 0 && lk > 0) lb = upper_safety(g, st, lk, rx, ry, rz);
              } else if constexpr (kStoreT) {
                for (int l = 0; l < L; ++l) level_distances(g, st, l, rx, ry, rz, u, v, w, os_l, os_s, b);
              } else {
                // frames accumulated level by level (T_0 = 0), as the descent built them
                double Tx = 0.0, Ty = 0.0, Tz = 0.0;
                for (int l = 0; l < L; ++l) {
                  const DUniv* U = g.univ + st.u(l);
                  const int kind_l = st.ukind(l), ia = st.a(l), ib = st.b(l), ic = st.c(l);
                  level_candidates(g, U, kind_l, ia, ib, ic, l, rx - Tx, ry - Ty, rz - Tz, u, v, w, os_l, os_s, b);
                  if (l + 1 < L) {
                    double tx, ty, tz;
                    level_translation(g, U, kind_l, ia, ib, ic, tx, ty, tz);
                    Tx = Tx + tx; Ty = Ty + ty; Tz = Tz + tz;
                  }
                }
              }
            }
            if (kSafe && mode == 1) {
              // merge with the deferred lower winner (levels [lk, L), evaluated after [0, lk) in the
              // canonical order: it wins only strictly).  F2: the runner-up of the union, via the
              // lower part's code (0: tie, 1: runner-up gap in (0, 1e-10], 2: larger)
              const double dl = sdl[slot];
              const int kl = sdesc[slot];
              const int code = (kl >> 30) & 3;
              if (dl < b.d) {
                near2 = code == 1 || (code == 2 && b.d - dl <= kFlagDist);
                b.d = dl;
                b.key = kl & 0x3FFFFFFF;
              } else {
                const double g2 = (dl < b.d2 ? dl : b.d2) - b.d;
                near2 = g2 > 0.0 && g2 <= kFlagDist;
              }
            } else {
              const double g2 = b.d2 - b.d;
              near2 = g2 > 0.0 && g2 <= kFlagDist;
              if (kSafe && mode == 0 && lk > 0) {
                // skip [0, lk) iff the stored bound covers them and exceeds the lower winner by the margins
                ssw = sss[slot];
                const double ss = static_cast<double>(__uint_as_float(ssw));
                defer = !(static_cast<int>(ssw & 7u) >= lk && (os_l < 0 || os_l >= lk) &&
                          ss * (1.0 - kSafeRel) > b.d + kSafeAbs);
              }
            }
            const double sig = ld(g.mc_st + mc);
            const double ds = b.d;
            const double dc = sig > 0.0 ? fdiv(tau, sig) : NT_INF;
            const double gc = fabs(dc - ds);
#ifdef NT_SAFETY_STATS
            // diagnostic build: cross_l4..l7 count mode-0 MOVEs with upper levels, deferrals, deferrals
            // for lack of a covering bound, U-ring MOVEs (the crossing total is then off)
            if (kSafe && mode == 0 && lk > 0) {
              atomicAdd(s_cnt + C_CBL0 + 4, 1u);
              if (defer) atomicAdd(s_cnt + C_CBL0 + 5, 1u);
              if (defer && static_cast<int>(ssw & 7u) < lk) atomicAdd(s_cnt + C_CBL0 + 6, 1u);
            }
            if (kSafe && mode == 1) atomicAdd(s_cnt + C_CBL0 + 7, 1u);
#endif
            if (defer) {
              // U ring: lower winner and its runner-up code; the slot's state is stored below unchanged
              const double g2l = b.d2 - b.d;
              const int code = g2l == 0.0 ? 0 : g2l <= kFlagDist ? 1 : 2;
              sdl[slot] = b.d;
              sdesc[slot] = (b.key & 0x3FFFFFFF) | (code << 30);
              outc = 6;
            } else {
            if (near2 || (gc > 0.0 && gc <= kFlagDist)) flags |= NT_F2;
            const int cell_before = TRACE ? ld(g.mc_cell + mc) : 0;
            if (ds == NT_INF && dc == NT_INF) {
              flags |= NT_F3;
              term = NT_T_LOST;
              outc = 5;
              emit<TRACE>(R, R.pid0 + sidx[slot], nseg, NT_EV_CROSS, -1, -1, cell_before, -1, 0.0, NT_T_LOST, flags);
            } else {
              const bool cross = ds < dc;
              const double s = cross ? ds : dc;
              atomicAdd(gl + mc, s);
              if (TALLY & 1) mesh_score(g, R.mesh, rx, ry, rz, u, v, w, s);
              if (TALLY & 2) atomicAdd(R.inst + instance_of(g, st, L), s);
              rx = rx + s * u; ry = ry + s * v; rz = rz + s * w;
              ++nseg;
              seg = true;
              if (TRACE) { sps[slot] = s; spcb[slot] = cell_before; }
              if (cross) {
                const double tt = tau - sig * s;
                tau = tt > 0.0 ? tt : 0.0;
                const int l = b.l(), jb = b.j();
                const bool csg_l = RTK != 0 ? (l == 0 || l == rg.K + 1) : st.ukind(l) == U_CSG;
                int meta = 0;
                int j = jb;
                if constexpr (RTK != 0) meta = l == 0 ? ld(g.surf_meta + jb) : 0;
                else j = winner_surface(g, csg_l, jb, meta);
                const int bc = l == 0 ? meta >> 4 : 0;
                if (bc == NT_BC_VACUUM) {
                  atomicAdd(s_exit + mc, 1u);
                  term = NT_T_LEAKED;
                  outc = 5;
                  lcross = -2;
                  emit<TRACE>(R, R.pid0 + sidx[slot], nseg - 1, NT_EV_LEAK, 0, j, cell_before, -1, s, NT_T_LEAKED, flags);
                } else if (bc == NT_BC_REFLECT) {
                  const int ax = meta & 15;
                  if (ax == 0) u = -u; else if (ax == 1) v = -v; else w = -w;
                  os_l = 0; os_s = j;
                  outc = 1;
                  emit<TRACE>(R, R.pid0 + sidx[slot], nseg - 1, NT_EV_REFLECT, 0, j, cell_before, cell_before, s,
                              NT_T_NONE, flags);
                } else {
                  atomicAdd(s_exit + mc, 1u);
                  lcross = l;
                  if (csg_l) {
                    sdesc[slot] = l | ((b.sense() ^ 1) << 4) | ((jb + 1) << 5);
                    os_l = l; os_s = j;
                    outc = 3;
                  } else {
                    sdesc[slot] = l | ((j + 1) << 5);
                    os_l = -1; os_s = -1;
                    outc = 4;
                  }
                  if (TRACE) { spl[slot] = static_cast<int8_t>(l); spj[slot] = j; }
                }
              } else {
                os_l = -1; os_s = -1;
                outc = 2;
              }
              if constexpr (kSafe) {
                // new safety of [0, cov): the bound at the pre-move point minus the path flown; a
                // reflection or a crossing at a covered level changes those levels: no bound
                uint32_t nw = 0;
                if (lk > 0 && outc != 5) {
                  const int cov = mode == 0 ? static_cast<int>(ssw & 7u) : lk;
                  const double base = mode == 0 ? static_cast<double>(__uint_as_float(ssw)) : lb;
                  if (!(outc == 1 || (cross && b.l() < cov))) nw = ss_pack(base - s, cov);
                }
                sss[slot] = nw;
              }
            }
            }   // not deferred
          }
          sx[slot] = rx; sy[slot] = ry; sz[slot] = rz;
          if (outc == 1) { su[slot] = u; sv[slot] = v; sw[slot] = w; }   // only a reflection turns the flight
          stau[slot] = tau;
          sflags[slot] = static_cast<uint8_t>(flags);
          snseg[slot] = nseg;
          sosl[slot] = static_cast<int8_t>(os_l);
          sos[slot] = os_s;
          if (outc == 5) finalize(slot, term);
        }
        // per-event counters (one shared atomic per warp and counter)
        warp_count(outc == 1, s_cnt + C_REFL, lane);   // collisions = segments - crossings - reflections (flush)
        if (lcross >= 0) atomicAdd(s_cnt + C_CBL0 + lcross, 1u);   // crossings = leaks + sum over levels (flush)
        // enqueue for the next event
        if constexpr (ASYNC) {
          // NR = 7: histories above the deepest level take the second set of rings (depth class)
          const bool cls = NR == 7 && ready && sL[slot] < maxd;
          push_all(ended_at_event || outc == 5 ? Q_F : outc == 1 ? Q_M : outc == 2 ? (cls ? Q_C2 : Q_C)
                   : outc == 3 ? (cls ? Q_DC2 : Q_DC) : outc == 4 ? Q_DA : (kSafe && outc == 6) ? QU : -1);
        } else {
          push(Q_M, outc == 1);
          push(Q_C, outc == 2);
          push(Q_DC, outc == 3);
          push(Q_DA, outc == 4);
          push(Q_F, outc == 5);
        }
      }
      if (ASYNC) base -= B;                       // ASYNC: keep claiming until the block is done
    }
    if (ASYNC) break;
    __syncthreads();
    // termination: no live history queued for the next round and no more pids
    if (QN(wr, Q_M) + QN(wr, Q_C) + QN(wr, Q_DC) + QN(wr, Q_DA) == 0 && s_flag[0]) break;
  }

  // ---- flush block tallies: exits / counters from shared memory, lengths from the block slice
  __syncthreads();
  if (tid == 0) {                        // crossings = leaks + non-leak crossings at every level
    unsigned int c = s_cnt[C_LEAK];
    for (int lv = 0; lv < kMaxDepth; ++lv) c += s_cnt[C_CBL0 + lv];
    s_cnt[C_CROSS] = c;
    s_cnt[C_COLL] = s_cnt[C_SEG] - c - s_cnt[C_REFL];  // every segment ends in one of the three
  }
  __syncthreads();
  flush_tallies(R, gl, s_exit, s_cnt, nmc, tid, B);
}

NT_DEV_END

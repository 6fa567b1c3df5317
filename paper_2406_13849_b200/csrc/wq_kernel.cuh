// Warp-queue generic tracker: warp-autonomous event queues (§2.3 event-based execution,
// P:420-434), the default scheduler.
//
// Each warp owns S particle slots in shared memory and keeps, in registers, one 64-bit mask per
// event queue: MOVE (distance_to_boundary + collide-or-cross + move + tally), COLLIDE
// (change_direction), DESCEND (find_cell / cross_surface descents, CSG-level and array-level
// separately so a warp descends one universe kind at a time) and FREE (slots to refill with new
// histories).  Every step the warp picks the fullest queue, gives lane i the i-th slot of it
// (__fns), processes up to 32 slots of ONE event type, and re-queues each slot by its outcome
// with two 32-bit REDUX.OR (__reduce_or_sync) per queue.  There is no block barrier: warps never
// wait for each other (the block-queue variant spent ~45% of its stalls at __syncthreads).
//
// The per-level universe stack keeps only indices (universe, cell / tile); the frame translation
// of every level is recomputed from them with exactly the descent's arithmetic, which halves the
// shared memory per slot and doubles the resident warps.  Results are bit-identical to the
// history scheduler and to the oracle.
#pragma once

NT_DEV_BEGIN

// Lane i receives the i-th slot of the concatenated queues m0, m1, m2 (in that order), encoded
// as slot | queue << 8, or -1 when i >= total: every set bit computes its rank with one popc and
// scatters its slot index into a per-warp buffer (__fns is emulated in software on sm_100a).
__device__ __forceinline__ int pick_slots(int* buf, int lane, uint64_t m0, uint64_t m1, uint64_t m2) {
  int base = 0;
  const uint64_t ms[3] = {m0, m1, m2};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const uint64_t m = ms[q];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      if ((m >> j) & 1ull) {
        const int r = base + __popcll(m & ((1ull << j) - 1ull));
        if (r < 32) buf[r] = j | (q << 8);
      }
    }
    base += __popcll(m);
  }
  __syncwarp();
  const int v = lane < base ? buf[lane] : -1;
  __syncwarp();
  return v;
}

__device__ __forceinline__ uint64_t warp_or64(bool pred, int slot) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (pred && slot < 32) ? (1u << slot) : 0u);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (pred && slot >= 32) ? (1u << (slot - 32)) : 0u);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ int popc64(uint64_t m) { return __popcll(m); }

constexpr int kWqSlots = 64;    // slots per warp
constexpr int kWqWarps = 4;     // warps per block

__host__ __device__ inline size_t wq_slot_bytes(int maxd, bool trace) {
  return (7 + (trace ? 1 : 0)) * 8 + (6 + (trace ? 2 : 0)) * 4 + 16 * (size_t)maxd + 3 + (trace ? 1 : 0);
}

constexpr size_t kWqPickBytes = 32 * 4;   // per-warp slot-pick buffer

size_t wq_smem_bytes(const DevGeom& g, bool trace) {
  size_t head = ((size_t)g.n_mc + kNC) * 4;
  head = (head + 15) & ~size_t(15);
  size_t warp = wq_slot_bytes(g.max_depth, trace) * kWqSlots + kWqPickBytes;
  warp = (warp + 15) & ~size_t(15);
  return head + warp * kWqWarps;
}

template <bool TRACE, bool STATES, int TALLY = 0>
__global__ void __launch_bounds__(kWqWarps * 32) k_track_wq(const DevGeom g, const KRun R) {
  constexpr int S = kWqSlots, W = kWqWarps, B = W * 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nmc = g.n_mc, maxd = g.max_depth;
  unsigned int* s_exit = reinterpret_cast<unsigned int*>(smem);
  unsigned int* s_cnt = s_exit + nmc;
  size_t head = ((size_t)nmc + kNC) * 4;
  head = (head + 15) & ~size_t(15);
  size_t wbytes = wq_slot_bytes(maxd, TRACE) * S + kWqPickBytes;
  wbytes = (wbytes + 15) & ~size_t(15);
  unsigned char* wb = smem + head + wbytes * warp;
  int* spick = reinterpret_cast<int*>(wb);
  wb += kWqPickBytes;
  // per-warp SoA slot storage
  double* sx = reinterpret_cast<double*>(wb);
  double* sy = sx + S; double* sz = sy + S; double* su = sz + S; double* sv = su + S; double* sw = sv + S;
  double* stau = sw + S;
  double* sps = stau + S;                               // TRACE only
  uint32_t* sidx = reinterpret_cast<uint32_t*>(sps + (TRACE ? S : 0));
  uint32_t* sepoch = sidx + S; uint32_t* snseg = sepoch + S;
  int32_t* smc = reinterpret_cast<int32_t*>(snseg + S);
  int32_t* sos = smc + S;
  int32_t* sdesc = sos + S;                             // pending descent: l0 | fsense<<4 | (fh+1)<<5
  int32_t* spj = sdesc + S;                             // TRACE only
  int32_t* spcb = spj + (TRACE ? S : 0);
  int32_t* sib = spcb + (TRACE ? S : 0);                // [maxd][4][S]
  uint8_t* sflags = reinterpret_cast<uint8_t*>(sib + 4 * maxd * S);
  uint8_t* sL = sflags + S;
  int8_t* sosl = reinterpret_cast<int8_t*>(sL + S);
  int8_t* spl = sosl + S;                               // TRACE only
  double* gl = R.slices + (size_t)blockIdx.x * nmc;

  for (int i = tid; i < nmc; i += B) s_exit[i] = 0u;
  for (int i = tid; i < kNC; i += B) s_cnt[i] = 0u;
  __syncthreads();

  const uint32_t max_seg = static_cast<uint32_t>(R.max_seg);
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
  };
  auto stack_of = [&](int slot) {
    Stack st;
    st.si = sib + slot;
    st.sT = nullptr;
    st.B = S;
    return st;
  };

  uint64_t mM = 0, mC = 0, mDC = 0, mDA = 0, mF = ~0ull;   // S == 64
  bool exhausted = false;

  for (;;) {
    const int nM = popc64(mM), nC = popc64(mC), nDC = popc64(mDC), nDA = popc64(mDA);
    const int nF = exhausted ? 0 : popc64(mF);
    const int nD = nDC + nDA + nF;
    if (nM + nC + nDC + nDA == 0 && nF == 0) break;
    // the fullest queue goes next (ties: MOVE, then DESCEND)
    const int stage = (nM >= nD && nM >= nC) ? 0 : (nD >= nC ? 1 : 2);

    if (stage == 1) {
      // ================= DESCEND (+ births) =================
      const int pk = pick_slots(spick, lane, mDC, mDA, exhausted ? 0ull : mF);
      const int slot = pk >= 0 ? (pk & 255) : 0, kind = pk >= 0 ? (pk >> 8) : 3;
      const unsigned bm = __ballot_sync(0xffffffffu, kind == 2);
      bool born = false, dead_slot = false;
      if (bm) {
        const int leader = __ffs(bm) - 1;
        unsigned long long b0 = 0;
        if (lane == leader) b0 = atomicAdd(R.counter, static_cast<unsigned long long>(__popc(bm)));
        b0 = __shfl_sync(0xffffffffu, b0, leader);
        if (kind == 2) {
          const unsigned long long id = b0 + __popc(bm & ((1u << lane) - 1u));
          if (id < R.n) { born = true; sidx[slot] = static_cast<uint32_t>(id); }
          else dead_slot = true;                             // no pids left: slot retires
        }
      }
      bool ok = false, done = false;
      if (kind == 0 || kind == 1 || born) {
        Stack st = stack_of(slot);
        double rx, ry, rz;
        uint32_t flags = 0;
        int L = 0, mc = 0;
        int l0 = 0, du = g.root, fh = -1, fsense = 0;
        double Tx = 0.0, Ty = 0.0, Tz = 0.0;
        if (born) {
          const uint64_t pid = R.pid0 + sidx[slot];
          double xa, xb, u, v, w;
          draw2(R.seed, pid, 0, 0, xa, xb);
          if (STATES) {
            const uint64_t id = sidx[slot];
            rx = R.states[id]; ry = R.states[R.n + id]; rz = R.states[2 * R.n + id];
            u = R.states[3 * R.n + id]; v = R.states[4 * R.n + id]; w = R.states[5 * R.n + id];
          } else {
            double xmu, xphi, xx, xy, xz, unused;
            draw2(R.seed, pid, 0, 1, xmu, xphi);
            draw2(R.seed, pid, 0, 2, xx, xy);
            draw2(R.seed, pid, 0, 3, xz, unused);
            rx = R.lo[0] + R.w[0] * xx;
            ry = R.lo[1] + R.w[1] * xy;
            rz = R.lo[2] + R.w[2] * xz;
            isotropic(xmu, xphi, u, v, w);
          }
          sx[slot] = rx; sy[slot] = ry; sz[slot] = rz;
          su[slot] = u; sv[slot] = v; sw[slot] = w;
          stau[slot] = -spec_log(xb);
          sepoch[slot] = 0; snseg[slot] = 0; sos[slot] = -1; sosl[slot] = -1;
          if (TRACE) spl[slot] = -2;
        } else {
          rx = sx[slot]; ry = sy[slot]; rz = sz[slot];
          flags = sflags[slot];
          const int dsc = sdesc[slot];
          l0 = dsc & 15;
          fsense = (dsc >> 4) & 1;
          fh = (dsc >> 5) - 1;
          // frame of level l0, recomputed top-down with the descent's arithmetic
          for (int l = 0; l < l0; ++l) {
            const DUniv* U = g.univ + st.u(l);
            double tx, ty, tz;
            level_translation(g, U, ld(&U->kind), st.a(l), st.b(l), st.c(l), tx, ty, tz);
            Tx = Tx + tx; Ty = Ty + ty; Tz = Tz + tz;
          }
          du = st.u(l0);
          if (kind == 1) {                                  // Alg. 6: tile +- 1, then the daughter
            const int j = fh;
            const DUniv* U = g.univ + du;
            const int uk = ld(&U->kind);
            int ta = st.a(l0), tb = st.b(l0), tc = st.c(l0);
            if (!kHex || uk == U_RECT) {
              const int dir = (j & 1) ? 1 : -1, ax = j >> 1;
              if (ax == 0) ta += dir; else if (ax == 1) tb += dir; else tc += dir;
            } else if (j < 6) {
              ta += (j == 0 || j == 5) ? 1 : ((j == 2 || j == 3) ? -1 : 0);
              tb += (j == 1 || j == 2) ? 1 : ((j == 4 || j == 5) ? -1 : 0);
            } else {
              tc += (j == 7) ? 1 : -1;
            }
            st.a(l0) = ta; st.b(l0) = tb; st.c(l0) = tc;
            double tx, ty, tz;
            du = array_daughter(g, U, uk, ta, tb, tc, tx, ty, tz);
            Tx = Tx + tx; Ty = Ty + ty; Tz = Tz + tz;
            l0 = l0 + 1;
            fh = -1;
            fsense = 0;
          }
        }
        ok = du >= 0 && descend<false>(g, st, l0, du, Tx, Ty, Tz, rx, ry, rz, fh, fsense, L, mc, flags);
        done = true;
        if (!ok) flags |= NT_F3;
        sflags[slot] = static_cast<uint8_t>(flags);
        if (ok) { sL[slot] = static_cast<uint8_t>(L); smc[slot] = mc; }
        if (TRACE) {
          const uint64_t pid = R.pid0 + sidx[slot];
          const int pl = spl[slot];
          if (pl == -2) {
            if (!ok) emit<TRACE>(R, pid, 0, NT_EV_CROSS, -1, -1, -1, -1, 0.0, NT_T_LOST, flags);
          } else {
            emit<TRACE>(R, pid, snseg[slot] - 1, NT_EV_CROSS, pl, spj[slot], spcb[slot], ok ? ld(g.mc_cell + mc) : -1,
                        sps[slot], ok ? NT_T_NONE : NT_T_LOST, flags);
          }
        }
        if (!ok) finalize(slot, NT_T_LOST);
      }
      const uint64_t taken = warp_or64(kind != 3, slot);
      mDC &= ~taken; mDA &= ~taken; mF &= ~taken;
      mM |= warp_or64(done && ok, slot);
      mF |= warp_or64(done && !ok, slot);
      exhausted = exhausted || __any_sync(0xffffffffu, dead_slot);
    } else if (stage == 0) {
      // ================= MOVE =================
      const int pk = pick_slots(spick, lane, mM, 0ull, 0ull);
      const bool valid = pk >= 0;
      const int slot = valid ? (pk & 255) : 0;
      int outc = 0, lcross = -1;
      bool seg = false;
      if (valid) {
        Stack st = stack_of(slot);
        double rx = sx[slot], ry = sy[slot], rz = sz[slot];
        double u = su[slot], v = sv[slot], w = sw[slot];
        double tau = stau[slot];
        uint32_t flags = sflags[slot], nseg = snseg[slot];
        const int L = sL[slot], mc = smc[slot];
        int os_l = sosl[slot], os_s = sos[slot];
        int term = NT_T_NONE;
        if (nseg >= max_seg) {
          flags |= NT_F3;
          term = NT_T_CAPPED;
          outc = 5;
          emit<TRACE>(R, R.pid0 + sidx[slot], nseg, NT_EV_COLLIDE, -1, -1, ld(g.mc_cell + mc), -1, 0.0,
                      NT_T_CAPPED, flags);
        } else {
          Best b;
          b.init();
          double Tx = 0.0, Ty = 0.0, Tz = 0.0;
          int kind_l = 0;                                    // universe kind of the crossing level
          for (int l = 0; l < L; ++l) {
            const DUniv* U = g.univ + st.u(l);
            const int kind = ld(&U->kind);
            const int ia = st.a(l), ib = st.b(l), ic = st.c(l);
            const int before = b.key;
            level_candidates(g, U, kind, ia, ib, ic, l, rx - Tx, ry - Ty, rz - Tz, u, v, w, os_l, os_s, b);
            if (b.key != before) kind_l = kind;
            if (l + 1 < L) {
              double tx, ty, tz;
              level_translation(g, U, kind, ia, ib, ic, tx, ty, tz);
              Tx = Tx + tx; Ty = Ty + ty; Tz = Tz + tz;
            }
          }
          const double sig = ld(g.mc_st + mc);
          const double ds = b.d;
          const double dc = sig > 0.0 ? fdiv(tau, sig) : NT_INF;
          const double g2 = b.d2 - ds, gc = fabs(dc - ds);
          if ((g2 > 0.0 && g2 <= kFlagDist) || (gc > 0.0 && gc <= kFlagDist)) flags |= NT_F2;
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
              int meta;
              const int j = winner_surface(g, kind_l == U_CSG, jb, meta);
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
                if (kind_l == U_CSG) {
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
          }
        }
        sx[slot] = rx; sy[slot] = ry; sz[slot] = rz;
        su[slot] = u; sv[slot] = v; sw[slot] = w;
        stau[slot] = tau;
        sflags[slot] = static_cast<uint8_t>(flags);
        snseg[slot] = nseg;
        sosl[slot] = static_cast<int8_t>(os_l);
        sos[slot] = os_s;
        if (outc == 5) finalize(slot, term);
      }
      warp_count(outc == 1, s_cnt + C_REFL, lane);
      if (lcross >= 0) atomicAdd(s_cnt + C_CBL0 + lcross, 1u);   // crossings = leaks + sum over levels (flush)
      mM &= ~warp_or64(valid, slot);
      mM |= warp_or64(outc == 1, slot);
      mC |= warp_or64(outc == 2, slot);
      mDC |= warp_or64(outc == 3, slot);
      mDA |= warp_or64(outc == 4, slot);
      mF |= warp_or64(outc == 5, slot);
    } else {
      // ================= COLLIDE =================
      const int pk = pick_slots(spick, lane, mC, 0ull, 0ull);
      const bool valid = pk >= 0;
      const int slot = valid ? (pk & 255) : 0;
      bool scat = false, absorbed = false;
      if (valid) {
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
          double xmu, xphi, u, v, w;
          draw2(R.seed, pid, epoch, 1, xmu, xphi);
          isotropic(xmu, xphi, u, v, w);
          su[slot] = u; sv[slot] = v; sw[slot] = w;
          stau[slot] = -spec_log(xb);
          scat = true;
          if (TRACE) emit<TRACE>(R, pid, snseg[slot] - 1, NT_EV_COLLIDE, -1, -1, cb, cb, sps[slot], NT_T_NONE, sflags[slot]);
        }
      }
      mC &= ~warp_or64(valid, slot);
      mM |= warp_or64(scat, slot);
      mF |= warp_or64(absorbed, slot);
    }
  }

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

// Rect-specialised comparison tracker (§3.3, Alg. 9-10): a fixed nesting
// root (axis box, or CZ annuli between a PZ pair) -> K rect arrays -> concentric-CZ pin, unrolled
// at compile time (the paper's template recursion) with non-polymorphic per-level code and the
// whole universe stack in registers.  It uses exactly the distance / location arithmetic of the
// generic tracker (nt_geom.cuh), so the two trackers are bit-identical on rect-shaped models
// (SURVEY pin P13) and their rate ratio isolates the cost of generality.
#pragma once

NT_DEV_BEGIN

template <int K, bool BOX, bool TRACE, bool STATES, int TALLY = 0>
__global__ void __launch_bounds__(256) k_track_rect(const DevGeom g, const RectGeom rg, const KRun R) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = blockDim.x, tid = threadIdx.x, lane = tid & 31;
  const int nmc = g.n_mc;
  unsigned int* s_cnt = reinterpret_cast<unsigned int*>(smem);
  unsigned int* s_exit = s_cnt + kNC;
  double* gl = R.slices + (size_t)blockIdx.x * nmc;   // per-block track-length tally (global)
  for (int i = tid; i < nmc; i += B) s_exit[i] = 0u;
  for (int i = tid; i < kNC; i += B) s_cnt[i] = 0u;
  __syncthreads();

  constexpr int KP = K + 1;          // pin level
  double rx = 0, ry = 0, rz = 0, u = 0, v = 0, w = 0, tau = 0;
  uint64_t pid = 0, idx = 0;
  uint32_t epoch = 0, flags = 0, nseg = 0, ncross = 0, ncoll = 0;
  int ann = 0;                       // CZ root: annulus (0 = core)
  int lu[K > 0 ? K : 1], li[K > 0 ? K : 1], lj[K > 0 ? K : 1], lk[K > 0 ? K : 1];
  double Tx[KP], Ty[KP], Tz[KP];     // frames of rect levels 1..K (index lv-1) and the pin (index K)
  int pin = 0, pa = 0, pin_u = 0;
  int mc = 0, os_l = -1, os_s = -1;
  bool core = true;                  // false while in an outer root annulus (material at level 0)
  int phase = 0, d_l0 = 0, d_fsid = -1, d_fsense = 0;
  int p_l = -1, p_j = -1, p_cb = -1;
  double p_s = 0;
  const uint32_t max_seg = static_cast<uint32_t>(R.max_seg);
  const double trx = ld(g.cell_tr + 3 * rg.root_fill_cell), try_ = ld(g.cell_tr + 3 * rg.root_fill_cell + 1),
               trz = ld(g.cell_tr + 3 * rg.root_fill_cell + 2);

  for (;;) {
    int term = NT_T_NONE;
    if (phase == 0) {
      const unsigned mask = __activemask();
      const int leader = __ffs(mask) - 1;
      const int rank = __popc(mask & ((1u << lane) - 1u));
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(R.counter, static_cast<unsigned long long>(__popc(mask)));
      base = __shfl_sync(mask, base, leader);
      idx = base + rank;
      if (idx >= R.n) break;
      pid = R.pid0 + idx;
      double xa, xb;
      draw2(R.seed, pid, 0, 0, xa, xb);
      const double xi_tau = xb;
      if (STATES) {
        rx = R.states[idx]; ry = R.states[R.n + idx]; rz = R.states[2 * R.n + idx];
        u = R.states[3 * R.n + idx]; v = R.states[4 * R.n + idx]; w = R.states[5 * R.n + idx];
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
      tau = -spec_log(xi_tau);
      epoch = 0; flags = 0; nseg = 0; ncross = 0; ncoll = 0; os_l = -1; os_s = -1;
      d_l0 = 0; d_fsid = -1; d_fsense = 0;
      p_l = -2;
      phase = 1;
    }
    if (phase == 1) {
      // ---- unrolled Alg. 9 find_cell from level d_l0 (forced sense at a CSG start level)
      bool ok = true;
      if (d_l0 == 0) {
        const int fsid = d_fsid, fsense = d_fsense;
        uint32_t nb = 0;
        if (BOX) {
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const int sid = rg.box_sid[k];
            int s;
            if (sid == fsid) {
              s = fsense;
            } else {
              const double f = surf_f(k >> 1, g.surf[sid].c, rx, ry, rz);
              s = f >= 0.0;
              if (fabs(f) <= ld(g.surf_tol + sid)) nb = 1u;
            }
            ok = ok && (s == ((k & 1) ? 0 : 1));
          }
          core = true;
        } else {
          int szl, szh;
          {
            const int sid = rg.zsid[0];
            if (sid == fsid) szl = fsense;
            else { const double f = surf_f(S_PZ, g.surf[sid].c, rx, ry, rz); szl = f >= 0.0; if (fabs(f) <= ld(g.surf_tol + sid)) nb = 1u; }
          }
          {
            const int sid = rg.zsid[1];
            if (sid == fsid) szh = fsense;
            else { const double f = surf_f(S_PZ, g.surf[sid].c, rx, ry, rz); szh = f >= 0.0; if (fabs(f) <= ld(g.surf_tol + sid)) nb = 1u; }
          }
          ok = szl == 1 && szh == 0;
          // annulus: first k with (k == 0 or inner sense POS) and outer sense NEG
          int found = -1, prev_pos = 1;
          uint32_t nb_in = 0, nb_prev = 0;
          for (int k = 0; k < rg.n_root_cells && found < 0; ++k) {
            const int sid = rg.root_sid[k];
            int s;
            uint32_t nbk = 0;
            if (sid == fsid) s = fsense;
            else { const double f = surf_f(S_CZ, g.surf[sid].c, rx, ry, rz); s = f >= 0.0; nbk = fabs(f) <= ld(g.surf_tol + sid); }
            if (prev_pos && s == 0) { found = k; nb_in = nb_prev | nbk; }
            prev_pos = s;
            nb_prev = nbk;
          }
          ok = ok && found >= 0;
          nb |= nb_in;
          ann = found < 0 ? 0 : found;
          core = ann == 0;
          if (ok && !core) mc = rg.root_mc[ann];
        }
        if (ok) flags |= nb;
        if (ok && core) {
          if (K > 0) { Tx[0] = 0.0 + trx; Ty[0] = 0.0 + try_; Tz[0] = 0.0 + trz; lu[0] = rg.root_univ_child; }
          else { Tx[K] = 0.0 + trx; Ty[K] = 0.0 + try_; Tz[K] = 0.0 + trz; pin_u = rg.root_univ_child; }
        }
      }
      // rect levels (Alg. 5 per level; translations accumulate as in the generic descent)
#pragma unroll
      for (int lv = 1; lv <= K; ++lv) {
        if (ok && core && lv >= d_l0) {
          const int q = lv - 1;
          const DUniv* U = g.univ + lu[q];
          const double x = rx - Tx[q], y = ry - Ty[q], z = rz - Tz[q];
          const double llx = ld(&U->d[0]), lly = ld(&U->d[1]), px = ld(&U->d[3]), py = ld(&U->d[4]);
          const int i = rect_index(llx, px, x), j = rect_index(lly, py, y);
          uint32_t nb = near_wall(llx, px, i, x) | near_wall(lly, py, j, y);
          int k = 0;
          if (!ld(&U->is2d)) {
            const double llz = ld(&U->d[2]), pz = ld(&U->d[5]);
            k = rect_index(llz, pz, z);
            nb |= near_wall(llz, pz, k, z);
          }
          flags |= nb;
          li[q] = i; lj[q] = j; lk[q] = k;
          double tx, ty, tz;
          const int dau = array_daughter(g, U, U_RECT, i, j, k, tx, ty, tz);
          if (dau < 0) ok = false;
          const int nq = lv < K ? lv : K;
          Tx[nq] = Tx[q] + tx; Ty[nq] = Ty[q] + ty; Tz[nq] = Tz[q] + tz;
          if (lv < K) lu[lv < K ? lv : 0] = dau; else pin_u = dau;
        }
      }
      // pin (concentric CZs): annulus = first k with (k == 0 or inner POS) and outer NEG
      if (ok && core) {
        pin = ld(rg.pin_of_univ + pin_u);
        const int off = ld(rg.pin_off + pin), ncz = ld(rg.pin_off + pin + 1) - off;
        const double x = rx - Tx[K], y = ry - Ty[K], z = rz - Tz[K];
        const int fsid = d_l0 == KP ? d_fsid : -1, fsense = d_fsense;
        int a = ncz, prev_pos = 1;
        uint32_t nb_prev = 0, nb_in = 0;
        for (int k = 0; k < ncz; ++k) {
          const int sid = ld(rg.pin_sid + off + k);
          int s;
          uint32_t nbk = 0;
          if (sid == fsid) s = fsense;
          else { const double f = surf_f(S_CZ, g.surf[sid].c, x, y, z); s = f >= 0.0; nbk = fabs(f) <= ld(g.surf_tol + sid); }
          if (prev_pos && s == 0) { a = k; nb_in = nb_prev | nbk; break; }
          prev_pos = s;
          nb_prev = nbk;
        }
        if (a == ncz) { nb_in = nb_prev; if (!prev_pos) ok = false; }
        flags |= nb_in;
        pa = a;
        mc = ld(rg.pin_mc + off + pin + a);
      }
      if (!ok) {
        flags |= NT_F3;
        term = NT_T_LOST;
        if (p_l == -2) emit<TRACE>(R, pid, 0, NT_EV_CROSS, -1, -1, -1, -1, 0.0, NT_T_LOST, flags);
        else emit<TRACE>(R, pid, nseg - 1, NT_EV_CROSS, p_l, p_j, p_cb, -1, p_s, NT_T_LOST, flags);
      } else {
        if (p_l != -2)
          emit<TRACE>(R, pid, nseg - 1, NT_EV_CROSS, p_l, p_j, p_cb, TRACE ? ld(g.mc_cell + mc) : 0, p_s,
                      NT_T_NONE, flags);
        phase = 2;
      }
    }
    if (phase == 2) {
      if (nseg >= max_seg) {
        flags |= NT_F3;
        term = NT_T_CAPPED;
        emit<TRACE>(R, pid, nseg, NT_EV_COLLIDE, -1, -1, ld(g.mc_cell + mc), -1, 0.0, NT_T_CAPPED, flags);
      } else {
        Best b;
        b.init();
        // level 0: the root cell's half-spaces in surface-id order
        if (BOX) {
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const int sid = rg.box_sid[k];
            const double d = surf_dist(k >> 1, (k & 1) ? 0 : 1, false, g.surf[sid].c, rx, ry, rz, u, v, w);
            b.consider(d, 0, sid, (k & 1) ? 0 : 1);
          }
        } else {
          {
            const int sid = rg.zsid[0];
            const double d = surf_dist(S_PZ, 1, false, g.surf[sid].c, rx, ry, rz, u, v, w);
            b.consider(d, 0, sid, 1);
          }
          {
            const int sid = rg.zsid[1];
            const double d = surf_dist(S_PZ, 0, false, g.surf[sid].c, rx, ry, rz, u, v, w);
            b.consider(d, 0, sid, 0);
          }
          if (ann > 0) {
            const int sid = rg.root_sid[ann - 1];
            const double d = surf_dist(S_CZ, 1, os_l == 0 && os_s == sid, g.surf[sid].c, rx, ry, rz, u, v, w);
            b.consider(d, 0, sid, 1);
          }
          {
            const int sid = rg.root_sid[ann];
            const double d = surf_dist(S_CZ, 0, os_l == 0 && os_s == sid, g.surf[sid].c, rx, ry, rz, u, v, w);
            b.consider(d, 0, sid, 0);
          }
        }
        if (core) {
#pragma unroll
          for (int lv = 1; lv <= K; ++lv) {
            const int q = lv - 1;
            const DUniv* U = g.univ + lu[q];
            const double x = rx - Tx[q], y = ry - Ty[q], z = rz - Tz[q];
            const int i = li[q], j = lj[q];
            if (u != 0.0) b.consider(rect_wall(ld(&U->d[0]), ld(&U->d[3]), i, x, u), lv, u > 0.0 ? 1 : 0, 0);
            if (v != 0.0) b.consider(rect_wall(ld(&U->d[1]), ld(&U->d[4]), j, y, v), lv, v > 0.0 ? 3 : 2, 0);
            if (!ld(&U->is2d) && w != 0.0)
              b.consider(rect_wall(ld(&U->d[2]), ld(&U->d[5]), lk[q], z, w), lv, w > 0.0 ? 5 : 4, 0);
          }
          // pin: inner cylinder (outside of it), then outer cylinder (inside of it)
          const int off = ld(rg.pin_off + pin), ncz = ld(rg.pin_off + pin + 1) - off;
          const double x = rx - Tx[K], y = ry - Ty[K], z = rz - Tz[K];
          if (pa > 0) {
            const int sid = ld(rg.pin_sid + off + pa - 1);
            const double d = surf_dist(S_CZ, 1, os_l == KP && os_s == sid, g.surf[sid].c, x, y, z, u, v, w);
            b.consider(d, KP, sid, 1);
          }
          if (pa < ncz) {
            const int sid = ld(rg.pin_sid + off + pa);
            const double d = surf_dist(S_CZ, 0, os_l == KP && os_s == sid, g.surf[sid].c, x, y, z, u, v, w);
            b.consider(d, KP, sid, 0);
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
          emit<TRACE>(R, pid, nseg, NT_EV_CROSS, -1, -1, cell_before, -1, 0.0, NT_T_LOST, flags);
        } else if (ds < dc) {
          const double s = ds;
          atomicAdd(gl + mc, s);
          if (TALLY & 1) mesh_score(g, R.mesh, rx, ry, rz, u, v, w, s);
          rx = rx + s * u; ry = ry + s * v; rz = rz + s * w;
          const double tt = tau - sig * s;
          tau = tt > 0.0 ? tt : 0.0;
          ++nseg;
          const int l = b.l(), j = b.j();
          const int meta = l == 0 ? ld(g.surf_meta + j) : 0;
          const int bc = meta >> 4;
          if (bc == NT_BC_VACUUM) {
            atomicAdd(s_exit + mc, 1u);
            ++ncross;
            term = NT_T_LEAKED;
            emit<TRACE>(R, pid, nseg - 1, NT_EV_LEAK, 0, j, cell_before, -1, s, NT_T_LEAKED, flags);
          } else if (bc == NT_BC_REFLECT) {
            const int ax = meta & 15;
            if (ax == 0) u = -u; else if (ax == 1) v = -v; else w = -w;
            os_l = 0; os_s = j;
            emit<TRACE>(R, pid, nseg - 1, NT_EV_REFLECT, 0, j, cell_before, cell_before, s, NT_T_NONE, flags);
          } else {
            atomicAdd(s_exit + mc, 1u);
            ++ncross;
            atomicAdd(s_cnt + C_CBL0 + l, 1u);
            p_l = l; p_j = j; p_cb = cell_before; p_s = s;
            phase = 1;
            if (l == 0 || l == KP) {            // CSG level: far side of surface j (Alg. 10)
              d_l0 = l; d_fsid = j; d_fsense = b.sense() ^ 1;
              os_l = l; os_s = j;
            } else {                            // rect level: tile +- 1 (Alg. 6), then its daughter
              d_fsid = -1; d_fsense = 0;
              os_l = -1; os_s = -1;
#pragma unroll
              for (int lv = 1; lv <= K; ++lv) {
                if (lv == l) {
                  const int q = lv - 1;
                  const int dir = (j & 1) ? 1 : -1, ax = j >> 1;
                  if (ax == 0) li[q] += dir; else if (ax == 1) lj[q] += dir; else lk[q] += dir;
                  double tx, ty, tz;
                  const int dau = array_daughter(g, g.univ + lu[q], U_RECT, li[q], lj[q], lk[q], tx, ty, tz);
                  const int nq = lv < K ? lv : K;
                  Tx[nq] = Tx[q] + tx; Ty[nq] = Ty[q] + ty; Tz[nq] = Tz[q] + tz;
                  if (lv < K) lu[lv < K ? lv : 0] = dau; else pin_u = dau;
                  if (dau < 0) {
                    flags |= NT_F3;
                    term = NT_T_LOST;
                    emit<TRACE>(R, pid, nseg - 1, NT_EV_CROSS, l, j, cell_before, -1, s, NT_T_LOST, flags);
                  }
                }
              }
              d_l0 = l + 1;
            }
          }
        } else {
          const double s = dc;
          atomicAdd(gl + mc, s);
          if (TALLY & 1) mesh_score(g, R.mesh, rx, ry, rz, u, v, w, s);
          rx = rx + s * u; ry = ry + s * v; rz = rz + s * w;
          ++nseg;
          ++ncoll;
          os_l = -1; os_s = -1;
          ++epoch;
          double xa, xb;
          draw2(R.seed, pid, epoch, 0, xa, xb);
          if (xa < ld(g.mc_pabs + mc)) {
            term = NT_T_ABSORBED;
            if (R.bank) bank_sites(g, R.bank, R.bank_n, mc, idx, xb, rx, ry, rz);
            emit<TRACE>(R, pid, nseg - 1, NT_EV_COLLIDE, -1, -1, cell_before, cell_before, s, NT_T_ABSORBED,
                        flags);
          } else {
            double xmu, xphi;
            draw2(R.seed, pid, epoch, 1, xmu, xphi);
            isotropic(xmu, xphi, u, v, w);
            tau = -spec_log(xb);
            emit<TRACE>(R, pid, nseg - 1, NT_EV_COLLIDE, -1, -1, cell_before, cell_before, s, NT_T_NONE, flags);
          }
        }
      }
      if (term == NT_T_NONE) continue;
    }
    phase = 0;
    atomicAdd(s_cnt + C_PART, 1u);
    atomicAdd(s_cnt + C_SEG, nseg);
    atomicAdd(s_cnt + C_CROSS, ncross);
    atomicAdd(s_cnt + C_COLL, ncoll);
    atomicAdd(s_cnt + C_REFL, nseg - ncross - ncoll);
    const int tcn = term == NT_T_ABSORBED ? C_ABS : term == NT_T_LEAKED ? C_LEAK : term == NT_T_LOST ? C_LOST : C_CAP;
    atomicAdd(s_cnt + tcn, 1u);
    if (flags) atomicAdd(s_cnt + C_FLAG, 1u);
    if (R.pflags) R.pflags[idx] = static_cast<uint8_t>(flags);
    if (R.pnseg) R.pnseg[idx] = nseg;
    if (R.pterm) R.pterm[idx] = static_cast<uint8_t>(term);
  }

  __syncthreads();
  flush_tallies(R, gl, s_exit, s_cnt, nmc, tid, B);
}

NT_DEV_END

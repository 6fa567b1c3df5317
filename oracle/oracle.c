/* ==========================================================================
 * ORACLE — test infrastructure, NOT product code.
 *
 * A plain, slow, brute-force CPU implementation of the nested-geometry
 * random walk of arXiv 2406.13849, written from the paper and the
 * readings O1-O26 of SURVEY.md §8(c) / DESIGN.md "Readings".  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no source, header, table or helper with the CUDA
 * path (paper_2406_13849_b200/csrc); the only shared input is the model spec
 * produced by workloads/models.py, marshalled by oracle/__init__.py.
 *
 * Plain definitions computed by brute force:
 *   - point location: every cell of a CSG universe is tested in id order
 *     (Alg. 3) level by level (Alg. 7); rect
 *     and hex indices are "the unique tile that owns the point" found by an
 *     explicit search (Alg. 5; hex reading O9);
 *   - distance to boundary: the minimum over every half-space of every
 *     level's current cell, plus the tile walls (Table 1).
 *   - mesh track-length tally (NEXT-2; reading M1 in DESIGN.md):
 *     every segment's [0, s] is cut at every mesh-plane crossing, the cut
 *     parameters are sorted, and each piece goes to the voxel that holds its
 *     midpoint (found by the same explicit search as a rect index).
 *   - per-instance (distributed-cell) tallies (NEXT-3; reading
 *     D1): the instance of a material cell is its position in the depth-first
 *     enumeration of all material-cell instances; counted by summing the leaves
 *     of every earlier sibling at every level.
 *   - fission source and k (NEXT-4, Alg. 1-2; reading F1): an
 *     absorption banks floor(nu Sigma_f / Sigma_a + xi) sites at the absorption
 *     point; the next cycle's source is drawn uniformly, with replacement, from
 *     the bank in (history, site) order.
 *   - non-uniform rect arrays (Alg. 5, P:513-525 and its footnote P:500-505):
 *     the tile is found by a linear scan over the mesh divisions (reading N1
 *     in DESIGN.md: index -1 below the first edge, n at or above the last).
 * Everything else follows Alg. 2 step by step: tau bookkeeping
 * (P:391-398), move/cross (Alg. 8; Alg. 6), collision
 * (P:399-409).
 *
 * Precision: IEEE fp64, compiled with -ffp-contract=off (no FMA).  The two
 * transcendental functions are the spec'd polynomial forms of DESIGN.md
 * reading R-T (orc_log, orc_sincos2pi), pinned against libm in the tests.
 *
 * Pins: tests/test_oracle_*.py (Philox KAT, U01, analytic distances, rect /
 * hex worked values, brute-force location, chord, volume, infinite medium,
 * nested==flat, additivity, closedness).  Absolute tallies of C1-C5 are
 * parity-unpinned by the paper and pinned only transitively.
 * ========================================================================== */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- constants */
enum { K_PX = 0, K_PY = 1, K_PZ = 2, K_PLANE = 3, K_CZ = 4, K_SPHERE = 5 };
enum { BC_NONE = 0, BC_VACUUM = 1, BC_REFLECT = 2 };
enum { U_CSG = 0, U_RECT = 1, U_HEX = 2 };
enum { FILL_MAT = 0, FILL_UNIV = 1 };
enum { POS = 1, NEG = 0 };
enum { F1 = 1, F2 = 2, F3 = 4 };
enum { EV_CROSS = 0, EV_REFLECT = 1, EV_LEAK = 2, EV_COLLIDE = 3 };
enum { T_NONE = 0, T_ABSORBED = 1, T_LEAKED = 2, T_LOST = 3, T_CAPPED = 4 };
/* counters block */
enum { C_PARTICLES, C_SEGMENTS, C_CROSSINGS, C_REFLECTIONS, C_LEAKS, C_COLLISIONS,
       C_ABSORPTIONS, C_LOST, C_CAPPED, C_FLAGGED, C_CBL0, NCOUNT = C_CBL0 + 8 };
/* distance-candidate evaluation kinds (F_alg) */
enum { E_AXIS = 0, E_PLANE = 1, E_CZ = 2, E_SPHERE = 3, E_RECT = 4, E_HEX = 5, NEVAL = 8 };

#define MAXD 8
#define FLAG_DIST 1e-10
static const double H_SQRT3_2 = 0.8660254037844386;   /* O9: nearest double to sqrt(3)/2 */

/* ---------------------------------------------------------------- model */
typedef struct { int kind, bc; double c[4]; double r2; double tol; } Surf;
typedef struct { double st, sa, pabs, nut; } Mat;   /* nut = nu Sigma_f / Sigma_a (F1) */
typedef struct {
    int uid, n, *sid, *sense;    /* half-spaces sorted by surface id */
    int fill_kind, fill;
    double tr[3];
    int mc;                      /* material-cell index (tally bin) or -1 */
} Cell;
typedef struct {
    int kind;
    /* CSG */
    int ncells, cap, *cells;
    /* RECT (O8); non-uniform (N1): e[a] = n[a]+1 increasing edges per axis, else NULL */
    double ll[3], p[3];
    int n[3], is2d;
    double *e[3];
    /* HEX (O9) */
    int orient, rings, nz;
    double C[2], pitch, pH, zlo, zp;
    double a1[2], a2[2], nrm[3][2];
    int *hexmap;                 /* (2R+1)^2 -> O9 order index or -1 */
    /* arrays */
    int *fill, nfill, outer;
} Univ;
typedef struct {
    int ns, nm, nc, nu, cs, cm, cc, cu;
    Surf *s; Mat *m; Cell *c; Univ *u;
    int root, finalized, n_mc, max_depth;
    /* superimposed Cartesian mesh (M1): voxel edges lo + i * d per axis, n[a] voxels */
    int mesh_on, mesh_n[3];
    double mesh_lo[3], mesh_d[3];
    long *leaves;                /* D1: material-cell instances below each universe (finalize) */
    int *mc_cell;                /* mc index -> global cell id */
} Model;

#define GROW(ptr, n, cap) do { if ((n) >= (cap)) { (cap) = (cap) ? 2 * (cap) : 16; \
    (ptr) = realloc((ptr), sizeof(*(ptr)) * (size_t)(cap)); } } while (0)

void *orc_model_new(void) { Model *m = calloc(1, sizeof(Model)); m->root = -1; return m; }

void orc_model_free(void *vm) {
    Model *m = vm;
    if (!m) return;
    for (int i = 0; i < m->nc; ++i) { free(m->c[i].sid); free(m->c[i].sense); }
    for (int i = 0; i < m->nu; ++i) {
        free(m->u[i].cells); free(m->u[i].fill); free(m->u[i].hexmap);
        for (int a = 0; a < 3; ++a) free(m->u[i].e[a]);
    }
    free(m->s); free(m->m); free(m->c); free(m->u); free(m->mc_cell); free(m->leaves); free(m);
}

int orc_add_surface(void *vm, int kind, const double *coef, int bc) {
    Model *m = vm;
    if (kind < 0 || kind > K_SPHERE) return -1;
    GROW(m->s, m->ns, m->cs);
    Surf *s = &m->s[m->ns];
    memset(s, 0, sizeof(*s));
    s->kind = kind; s->bc = bc;
    int nco = kind <= K_PZ ? 1 : (kind == K_CZ ? 3 : 4);
    for (int i = 0; i < nco; ++i) s->c[i] = coef[i];
    /* O3: R*R computed once; O16: flag tolerance 1e-10 x |grad f| scale */
    if (kind == K_CZ) { s->r2 = s->c[2] * s->c[2]; s->tol = FLAG_DIST * (2.0 * s->c[2]); }
    else if (kind == K_SPHERE) { s->r2 = s->c[3] * s->c[3]; s->tol = FLAG_DIST * (2.0 * s->c[3]); }
    else if (kind == K_PLANE) {
        s->tol = FLAG_DIST * sqrt((s->c[0] * s->c[0] + s->c[1] * s->c[1]) + s->c[2] * s->c[2]);
    } else s->tol = FLAG_DIST;
    return m->ns++;
}

int orc_add_material(void *vm, double st, double sa) {
    Model *m = vm;
    GROW(m->m, m->nm, m->cm);
    m->m[m->nm].st = st; m->m[m->nm].sa = sa;
    m->m[m->nm].pabs = st > 0.0 ? sa / st : 0.0;     /* O14: IEEE division, once */
    m->m[m->nm].nut = 0.0;
    return m->nm++;
}

/* F1: one-group nu Sigma_f of a material (>= 0; > 0 needs Sigma_a > 0).  Stored as the expected
 * number of sites per absorption, nu Sigma_f / Sigma_a (IEEE division, once). */
int orc_set_fission(void *vm, int mat, double nusf) {
    Model *m = vm;
    if (mat < 0 || mat >= m->nm || !(nusf >= 0.0) || !isfinite(nusf)) return -1;
    if (nusf > 0.0 && !(m->m[mat].sa > 0.0)) return -1;
    m->m[mat].nut = nusf > 0.0 ? nusf / m->m[mat].sa : 0.0;
    return 0;
}

/* F1: maximum number of sites one absorption can bank: floor(max nut) + 1 */
int orc_max_sites(void *vm) {
    Model *m = vm;
    double mx = 0.0;
    for (int i = 0; i < m->nm; ++i) if (m->m[i].nut > mx) mx = m->m[i].nut;
    return (int)floor(mx) + 1;
}

static int new_univ(Model *m, int kind) {
    GROW(m->u, m->nu, m->cu);
    memset(&m->u[m->nu], 0, sizeof(Univ));
    m->u[m->nu].kind = kind;
    m->u[m->nu].outer = -1;
    return m->nu++;
}

int orc_add_csg_universe(void *vm) { return new_univ(vm, U_CSG); }

int orc_add_cell(void *vm, int uid, const int *hs, int n, int fill_kind, int fill, const double *tr) {
    Model *m = vm;
    if (uid < 0 || uid >= m->nu || m->u[uid].kind != U_CSG || n < 0) return -1;   /* n == 0: all space */
    GROW(m->c, m->nc, m->cc);
    Cell *c = &m->c[m->nc];
    memset(c, 0, sizeof(*c));
    c->uid = uid; c->n = n; c->fill_kind = fill_kind; c->fill = fill; c->mc = -1;
    c->sid = malloc(sizeof(int) * (size_t)(n + 1));
    c->sense = malloc(sizeof(int) * (size_t)(n + 1));
    for (int i = 0; i < n; ++i) {
        int h = hs[i];
        c->sid[i] = (h > 0 ? h : -h) - 1;
        c->sense[i] = h > 0 ? POS : NEG;
    }
    /* O13: canonical candidate order = half-spaces sorted by surface id (insertion sort) */
    for (int i = 1; i < n; ++i)
        for (int j = i; j > 0 && c->sid[j - 1] > c->sid[j]; --j) {
            int t = c->sid[j]; c->sid[j] = c->sid[j - 1]; c->sid[j - 1] = t;
            t = c->sense[j]; c->sense[j] = c->sense[j - 1]; c->sense[j - 1] = t;
        }
    for (int i = 0; i < 3; ++i) c->tr[i] = tr ? tr[i] : 0.0;
    Univ *u = &m->u[uid];
    GROW(u->cells, u->ncells, u->cap);
    u->cells[u->ncells++] = m->nc;
    return m->nc++;
}

int orc_add_rect(void *vm, const double *ll, const double *p, const int *shape, const int *fill, int outer) {
    Model *m = vm;
    int id = new_univ(m, U_RECT);
    Univ *u = &m->u[id];
    for (int i = 0; i < 3; ++i) { u->ll[i] = ll[i]; u->p[i] = p[i]; u->n[i] = shape[i]; }
    u->is2d = p[2] == 0.0;
    if (u->is2d) u->n[2] = 1;
    u->nfill = u->n[0] * u->n[1] * u->n[2];
    u->fill = malloc(sizeof(int) * (size_t)u->nfill);
    memcpy(u->fill, fill, sizeof(int) * (size_t)u->nfill);
    u->outer = outer;
    return id;
}

/* Non-uniform rect array (Alg. 5 binary-search lattices): ne[a] edges per axis
 * (ne[2] == 0: 2-D), concatenated x, y, z in `edges`, strictly increasing.  Returns -1 on bad
 * edges. */
int orc_add_rect_edges(void *vm, const double *edges, const int *ne, const int *fill, int outer) {
    Model *m = vm;
    if (ne[0] < 2 || ne[1] < 2 || (ne[2] != 0 && ne[2] < 2)) return -1;
    int off = 0;
    for (int a = 0; a < 3; ++a) {
        for (int i = 1; i < ne[a]; ++i)
            if (!(edges[off + i - 1] < edges[off + i]) || !isfinite(edges[off + i])) return -1;
        off += ne[a];
    }
    int id = new_univ(m, U_RECT);
    Univ *u = &m->u[id];
    off = 0;
    for (int a = 0; a < 3; ++a) {
        u->n[a] = ne[a] > 0 ? ne[a] - 1 : 1;
        u->ll[a] = 0.0; u->p[a] = 0.0;
        if (ne[a] > 0) {
            u->e[a] = malloc(sizeof(double) * (size_t)ne[a]);
            memcpy(u->e[a], edges + off, sizeof(double) * (size_t)ne[a]);
        }
        off += ne[a];
    }
    u->is2d = ne[2] == 0;
    u->nfill = u->n[0] * u->n[1] * u->n[2];
    u->fill = malloc(sizeof(int) * (size_t)u->nfill);
    memcpy(u->fill, fill, sizeof(int) * (size_t)u->nfill);
    u->outer = outer;
    return id;
}

int orc_add_hex(void *vm, int orient, const double *C, double pitch, int rings, double zlo, double zp,
                int nz, const int *fill, int outer) {
    Model *m = vm;
    int id = new_univ(m, U_HEX);
    Univ *u = &m->u[id];
    u->orient = orient; u->C[0] = C[0]; u->C[1] = C[1]; u->pitch = pitch; u->rings = rings;
    u->zlo = zlo; u->zp = zp; u->nz = zp == 0.0 ? 0 : nz;
    u->pH = pitch * H_SQRT3_2;          /* O9: p*H rounded once */
    const double H = H_SQRT3_2;
    if (orient == 0) {   /* POINTY: a1=(p,0), a2=(p/2, pH); normals at 0,60,120 deg */
        u->a1[0] = pitch; u->a1[1] = 0.0; u->a2[0] = pitch * 0.5; u->a2[1] = u->pH;
        u->nrm[0][0] = 1.0;  u->nrm[0][1] = 0.0;
        u->nrm[1][0] = 0.5;  u->nrm[1][1] = H;
        u->nrm[2][0] = -0.5; u->nrm[2][1] = H;
    } else {             /* FLAT: a1=(pH, p/2), a2=(0,p); normals at 30,90,150 deg */
        u->a1[0] = u->pH; u->a1[1] = pitch * 0.5; u->a2[0] = 0.0; u->a2[1] = pitch;
        u->nrm[0][0] = H;  u->nrm[0][1] = 0.5;
        u->nrm[1][0] = 0.0; u->nrm[1][1] = 1.0;
        u->nrm[2][0] = -H; u->nrm[2][1] = 0.5;
    }
    int R = rings - 1, W = 2 * R + 1, ntile = 0;
    u->hexmap = malloc(sizeof(int) * (size_t)(W * W));
    for (int r = -R; r <= R; ++r)          /* O9 fill order: r ascending, then q ascending */
        for (int q = -R; q <= R; ++q) {
            int a = abs(q), b = abs(r), c = abs(q + r);
            int d = a > b ? a : b; d = d > c ? d : c;
            u->hexmap[(r + R) * W + (q + R)] = d <= R ? ntile++ : -1;
        }
    u->nfill = ntile * (u->nz > 0 ? u->nz : 1);
    u->fill = malloc(sizeof(int) * (size_t)u->nfill);
    memcpy(u->fill, fill, sizeof(int) * (size_t)u->nfill);
    u->outer = outer;
    return id;
}

int orc_set_root(void *vm, int uid) { ((Model *)vm)->root = uid; return 0; }

/* depth of the deepest material cell below universe u (levels counted from u = 1) */
static int depth_of(Model *m, int u, int guard) {
    if (guard > 32) return 1000;
    Univ *U = &m->u[u];
    int best = 0;
    if (U->kind == U_CSG) {
        for (int i = 0; i < U->ncells; ++i) {
            Cell *c = &m->c[U->cells[i]];
            int d = c->fill_kind == FILL_MAT ? 1 : 1 + depth_of(m, c->fill, guard + 1);
            if (d > best) best = d;
        }
    } else {
        for (int i = 0; i <= U->nfill; ++i) {
            int f = i < U->nfill ? U->fill[i] : U->outer;
            if (f < 0) continue;
            int d = 1 + depth_of(m, f, guard + 1);
            if (d > best) best = d;
        }
    }
    return best;
}

/* D1: number of material-cell instances below universe u in the depth-first enumeration: a CSG
 * universe's cells in id order (a material cell is one instance, a fill cell contributes its
 * universe's instances), an array's tiles in fill order and then its outer universe once. */
static long leaves_of(Model *m, int u) {
    if (m->leaves[u] >= 0) return m->leaves[u];
    const Univ *U = &m->u[u];
    long n = 0;
    if (U->kind == U_CSG) {
        for (int i = 0; i < U->ncells; ++i) {
            const Cell *c = &m->c[U->cells[i]];
            n += c->fill_kind == FILL_MAT ? 1 : leaves_of(m, c->fill);
        }
    } else {
        for (int i = 0; i < U->nfill; ++i) n += leaves_of(m, U->fill[i]);
        if (U->outer >= 0) n += leaves_of(m, U->outer);
    }
    m->leaves[u] = n;
    return n;
}

int orc_finalize(void *vm) {
    Model *m = vm;
    if (m->root < 0 || m->root >= m->nu) return -1;
    for (int i = 0; i < m->nc; ++i) {
        Cell *c = &m->c[i];
        for (int k = 0; k < c->n; ++k) if (c->sid[k] < 0 || c->sid[k] >= m->ns) return -2;
        if (c->fill_kind == FILL_MAT && (c->fill < 0 || c->fill >= m->nm)) return -3;
        if (c->fill_kind == FILL_UNIV && (c->fill < 0 || c->fill >= m->nu)) return -4;
    }
    for (int i = 0; i < m->nu; ++i) {
        Univ *u = &m->u[i];
        if (u->kind != U_CSG)
            for (int k = 0; k <= u->nfill; ++k) {
                int f = k < u->nfill ? u->fill[k] : u->outer;
                if (f < -1 || f >= m->nu || (k < u->nfill && f < 0)) return -5;
            }
    }
    m->max_depth = depth_of(m, m->root, 0);
    if (m->max_depth > MAXD) return -6;
    free(m->leaves);
    m->leaves = malloc(sizeof(long) * (size_t)(m->nu + 1));
    for (int i = 0; i < m->nu; ++i) m->leaves[i] = -1;
    for (int i = 0; i < m->nu; ++i) leaves_of(m, i);
    /* material cells get dense tally indices in global cell-id order (O20) */
    free(m->mc_cell);
    m->mc_cell = malloc(sizeof(int) * (size_t)(m->nc + 1));
    m->n_mc = 0;
    for (int i = 0; i < m->nc; ++i)
        if (m->c[i].fill_kind == FILL_MAT) { m->c[i].mc = m->n_mc; m->mc_cell[m->n_mc++] = i; }
    m->finalized = 1;
    return 0;
}

int orc_n_material_cells(void *vm) { return ((Model *)vm)->n_mc; }
int orc_max_depth(void *vm) { return ((Model *)vm)->max_depth; }
int orc_out_len(void *vm) { return 2 * ((Model *)vm)->n_mc + NCOUNT; }
int orc_material_cell_ids(void *vm, int *out) {
    Model *m = vm;
    for (int i = 0; i < m->n_mc; ++i) out[i] = m->mc_cell[i];
    return m->n_mc;
}
int orc_cell_material(void *vm, int cell) {
    Model *m = vm;
    return m->c[cell].fill_kind == FILL_MAT ? m->c[cell].fill : -1;
}

/* ======================================================================
 * RNG: Philox4x32-10 (Random123 constants), U01 (O17/P2)
 * ====================================================================== */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

double orc_u01(uint32_t h, uint32_t l) {
    uint64_t k = ((((uint64_t)h) << 32) | (uint64_t)l) >> 12;
    return ((double)k + 0.5) * 0x1p-52;
}

/* draw block b of epoch e for particle pid: (xi_A, xi_B) */
static void draw(uint64_t seed, uint64_t pid, uint32_t epoch, uint32_t block, double *xa, double *xb) {
    uint32_t ctr[4] = {(uint32_t)pid, (uint32_t)(pid >> 32), epoch, block};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox(ctr, key, o);
    *xa = orc_u01(o[0], o[1]);
    *xb = orc_u01(o[2], o[3]);
}

/* ======================================================================
 * Spec'd transcendentals (reading R-T).  Plain polynomial forms,
 * IEEE ops only, so the CUDA path can reproduce them bit-for-bit.
 * ====================================================================== */
double orc_log(double x) {
    /* x = m 2^e, m in [0.5,1); move m into [sqrt(1/2), sqrt(2)) */
    int e;
    double m = frexp(x, &e);
    if (m < 0.7071067811865476) { m = m * 2.0; e = e - 1; }
    double f = m - 1.0;
    double s = f / (2.0 + f);
    double z = s * s;
    /* log(m) = 2 atanh(s) = 2s (1 + z/3 + z^2/5 + ... + z^11/23) */
    double p = 1.0 / 23.0;
    for (int k = 10; k >= 0; --k) p = p * z + 1.0 / (double)(2 * k + 1);
    double lm = (2.0 * s) * p;
    double ed = (double)e;
    const double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
    return ed * LN2_HI + (ed * LN2_LO + lm);
}

/* cos(2 pi xi), sin(2 pi xi) for xi in (0,1): quadrant reduction of 4 xi (exact) then
 * Taylor series on [0, pi/4]. */
void orc_sincos2pi(double xi, double *co, double *si) {
    double x = xi * 4.0;
    int q = (int)floor(x);
    double f = x - (double)q;
    int swap = f > 0.5;
    double g = swap ? 1.0 - f : f;
    double a = g * 1.5707963267948966;
    double z = a * a;
    double fact[20];
    fact[0] = 1.0;
    for (int k = 1; k < 20; ++k) fact[k] = fact[k - 1] * (double)k;
    /* sin: a + a z (S1 + z (S2 + ... + z S9)),  S_k = (-1)^k / (2k+1)! */
    double ps = 1.0 / fact[19];
    ps = -ps;                                   /* S9 = -1/19! */
    for (int k = 8; k >= 1; --k) {
        double sk = 1.0 / fact[2 * k + 1];
        if (k & 1) sk = -sk;
        ps = ps * z + sk;
    }
    double sa = a + (a * z) * ps;
    /* cos: 1 + z (C1 + z (C2 + ... + z C9)),  C_k = (-1)^k / (2k)! */
    double pc = 1.0 / fact[18];
    pc = -pc;                                   /* C9 = -1/18! */
    for (int k = 8; k >= 1; --k) {
        double ck = 1.0 / fact[2 * k];
        if (k & 1) ck = -ck;
        pc = pc * z + ck;
    }
    double ca = 1.0 + z * pc;
    double C = swap ? sa : ca, S = swap ? ca : sa;   /* cos, sin of f*pi/2 */
    switch (q & 3) {
        case 0: *co = C; *si = S; break;
        case 1: *co = -S; *si = C; break;
        case 2: *co = -C; *si = -S; break;
        default: *co = S; *si = -C; break;
    }
}

/* O15 isotropic direction */
static void iso(double xmu, double xphi, double om[3]) {
    double mu = 2.0 * xmu - 1.0;
    double t = 1.0 - mu * mu;
    double s = sqrt(t > 0.0 ? t : 0.0);
    double c, sn;
    orc_sincos2pi(xphi, &c, &sn);
    om[0] = s * c; om[1] = s * sn; om[2] = mu;
}

/* ======================================================================
 * Surfaces: implicit function (O3), sense (O4), cell-aware distance (O11)
 * ====================================================================== */
static double surf_f(const Surf *s, const double r[3]) {
    switch (s->kind) {
        case K_PX: return r[0] - s->c[0];
        case K_PY: return r[1] - s->c[0];
        case K_PZ: return r[2] - s->c[0];
        case K_PLANE: return ((s->c[0] * r[0] + s->c[1] * r[1]) + s->c[2] * r[2]) - s->c[3];
        case K_CZ: {
            double dx = r[0] - s->c[0], dy = r[1] - s->c[1];
            return (dx * dx + dy * dy) - s->r2;
        }
        default: {
            double dx = r[0] - s->c[0], dy = r[1] - s->c[1], dz = r[2] - s->c[2];
            return ((dx * dx + dy * dy) + dz * dz) - s->r2;
        }
    }
}

static int sense_of(double f) { return f >= 0.0 ? POS : NEG; }   /* O4 */

static double clamp0(double d) { return d > 0.0 ? d : 0.0; }

/* forward distance to leave half-space (s, sigma) from local r along om (O11);
 * os: particle is logically on this surface (quadric c := 0). INFINITY = no exit. */
static double surf_dist(const Surf *s, int sigma, int os, const double r[3], const double om[3],
                        uint64_t *ev) {
    switch (s->kind) {
        case K_PX: case K_PY: case K_PZ: {
            int a = s->kind;
            double u = om[a];
            if (u == 0.0) return INFINITY;
            if (!((sigma == NEG && u > 0.0) || (sigma == POS && u < 0.0))) return INFINITY;
            if (ev) ev[E_AXIS]++;
            return clamp0((s->c[0] - r[a]) / u);
        }
        case K_PLANE: {
            double sd = (s->c[0] * om[0] + s->c[1] * om[1]) + s->c[2] * om[2];
            if (sd == 0.0) return INFINITY;
            if (!((sigma == NEG && sd > 0.0) || (sigma == POS && sd < 0.0))) return INFINITY;
            if (ev) ev[E_PLANE]++;
            double fr = (s->c[0] * r[0] + s->c[1] * r[1]) + s->c[2] * r[2];
            return clamp0((s->c[3] - fr) / sd);
        }
        case K_CZ: case K_SPHERE: {
            double a, k, c, q;
            if (s->kind == K_CZ) {
                double dx = r[0] - s->c[0], dy = r[1] - s->c[1];
                a = om[0] * om[0] + om[1] * om[1];
                if (a == 0.0) return INFINITY;
                k = dx * om[0] + dy * om[1];
                c = os ? 0.0 : (dx * dx + dy * dy) - s->r2;
                q = k * k - a * c;
            } else {
                double dx = r[0] - s->c[0], dy = r[1] - s->c[1], dz = r[2] - s->c[2];
                a = 1.0;
                k = (dx * om[0] + dy * om[1]) + dz * om[2];
                c = os ? 0.0 : ((dx * dx + dy * dy) + dz * dz) - s->r2;
                q = k * k - c;
            }
            if (sigma == NEG) {
                if (ev) ev[s->kind == K_CZ ? E_CZ : E_SPHERE]++;
                if (q < 0.0) q = 0.0;
                double d = k <= 0.0 ? (-k + sqrt(q)) / a : -c / (k + sqrt(q));
                return clamp0(d);
            } else {
                if (k >= 0.0) return INFINITY;
                if (q < 0.0) return INFINITY;
                if (ev) ev[s->kind == K_CZ ? E_CZ : E_SPHERE]++;
                return clamp0(c / (-k + sqrt(q)));
            }
        }
    }
    return INFINITY;
}

/* ======================================================================
 * Single-universe location (brute force).  Result of a level.
 * ====================================================================== */
typedef struct {
    int u;            /* universe id at this level */
    int cell;         /* CSG: global cell id */
    int i, j, k;      /* RECT: tile ijk; HEX: q, r, kz */
    double T[3];      /* O6: accumulated translation of this level's frame */
} Level;

typedef struct { int daughter; int mc; int mat; double t[3]; } LocOut;

static void local_pos(const double r[3], const double T[3], double out[3]) {
    out[0] = r[0] - T[0]; out[1] = r[1] - T[1]; out[2] = r[2] - T[2];
}

/* Alg. 3 "cell contains pos" with an optional logically forced sense (O9') */
static int cell_contains(const Model *m, const Cell *c, const double rl[3], int fsid, int fsense) {
    for (int h = 0; h < c->n; ++h) {
        int sn;
        if (c->sid[h] == fsid) sn = fsense;
        else sn = sense_of(surf_f(&m->s[c->sid[h]], rl));
        if (sn != c->sense[h]) return 0;
    }
    return 1;
}

static int cell_near(const Model *m, const Cell *c, const double rl[3], int skip_sid) {
    for (int h = 0; h < c->n; ++h) {
        if (c->sid[h] == skip_sid) continue;
        const Surf *s = &m->s[c->sid[h]];
        if (fabs(surf_f(s, rl)) <= s->tol) return 1;     /* O16 F1 */
    }
    return 0;
}

/* rect edge e(i) = LL + i p (O8, mul then add) */
static double edge(double ll, double p, int i) { return ll + (double)i * p; }

/* O8: the unique i with e(i) <= x < e(i+1), found by an explicit search */
static int rect_axis_index(double ll, double p, double x) {
    int i = (int)floor((x - ll) / p);              /* starting guess only */
    while (!(edge(ll, p, i) <= x)) i--;
    while (!(x < edge(ll, p, i + 1))) i++;
    return i;
}
static int rect_axis_index_u(const Univ *U, int a, double x) { return rect_axis_index(U->ll[a], U->p[a], x); }

/* Reading N1, non-uniform axis with edges e[0..n]: tile i spans [E(i), E(i+1)) with
 * E(i) = e[i] for 0 <= i <= n, E(-1) = -inf, E(n+1) = +inf; so tile -1 is the slab below e[0]
 * and tile n the slab at or above e[n] (both `outer`).  Tile centre (the daughter translation):
 * (e[i] + e[i+1]) * 0.5 inside, e[0] for tile -1, e[n] for tile n. */
static double nu_edge(const Univ *U, int a, int i) {
    if (i < 0) return -INFINITY;
    if (i > U->n[a]) return INFINITY;
    return U->e[a][i];
}
static int nu_index(const Univ *U, int a, double x) {
    for (int i = -1; i <= U->n[a]; ++i)                    /* linear scan: the definition */
        if (nu_edge(U, a, i) <= x && x < nu_edge(U, a, i + 1)) return i;
    return U->n[a];                                         /* not reached for finite x */
}
static double nu_centre(const Univ *U, int a, int i) {
    if (i < 0) return U->e[a][0];
    if (i >= U->n[a]) return U->e[a][U->n[a]];
    return (U->e[a][i] + U->e[a][i + 1]) * 0.5;
}
/* tile edge / centre of rect axis a, uniform or not */
static double tile_edge(const Univ *U, int a, int i) {
    return U->e[a] ? nu_edge(U, a, i) : edge(U->ll[a], U->p[a], i);
}
static int tile_index(const Univ *U, int a, double x) {
    return U->e[a] ? nu_index(U, a, x) : rect_axis_index_u(U, a, x);
}
static double tile_centre(const Univ *U, int a, int i) {
    return U->e[a] ? nu_centre(U, a, i) : U->ll[a] + ((double)i + 0.5) * U->p[a];
}

/* hex s-space (reading O9): s_k = n_k . (x - C), the signed distance along face normal k in the
 * lattice frame; tile (q, r) spans p (m_k - 1/2) <= s_k < p (m_k + 1/2) */
static void hex_s(const Univ *U, const double rl[3], double t[3]) {
    double x = rl[0] - U->C[0], y = rl[1] - U->C[1];
    for (int k = 0; k < 3; ++k) t[k] = U->nrm[k][0] * x + U->nrm[k][1] * y;
}
static void hex_m(int q, int r, double mm[3]) {
    mm[0] = (double)q + (double)r * 0.5;
    mm[1] = (double)q * 0.5 + (double)r;
    mm[2] = -((double)q * 0.5) + (double)r * 0.5;
}
static int hex_owns(const Univ *U, int q, int r, const double t[3]) {
    double mm[3];
    hex_m(q, r, mm);
    for (int k = 0; k < 3; ++k)
        if (!(U->pitch * (mm[k] - 0.5) <= t[k] && t[k] < U->pitch * (mm[k] + 0.5))) return 0;
    return 1;
}
/* cube rounding of fractional axial coords: the GPU-visible fallback tile (O9) */
static void hex_cube_round(const Univ *U, const double rl[3], int *qo, int *ro) {
    double x = rl[0] - U->C[0], y = rl[1] - U->C[1];
    double qf, rf;
    if (U->orient == 0) { rf = y / U->pH; qf = (x - rf * (U->pitch * 0.5)) / U->pitch; }
    else { qf = x / U->pH; rf = (y - qf * (U->pitch * 0.5)) / U->pitch; }
    double sf = -qf - rf;
    double qr = round(qf), rr = round(rf), sr = round(sf);
    double dq = fabs(qr - qf), dr = fabs(rr - rf), ds = fabs(sr - sf);
    if (dq > dr && dq > ds) qr = -rr - sr;
    else if (dr > ds) rr = -qr - sr;
    *qo = (int)qr; *ro = (int)rr;
}

/* Locate rl in universe u at one level. Returns 1 on success (O6-O10).
 * fsid/fsense: forced sense (CSG crossing, O9'), fsid = -1 for none. *near |= F1 bits. */
static int locate(const Model *m, int u, const double rl[3], int fsid, int fsense, Level *L,
                  LocOut *o, int *near) {
    const Univ *U = &m->u[u];
    L->u = u; L->cell = -1; L->i = L->j = L->k = 0;
    o->t[0] = o->t[1] = o->t[2] = 0.0;
    if (U->kind == U_CSG) {
        for (int i = 0; i < U->ncells; ++i) {                 /* Alg. 3: every cell, id order */
            const Cell *c = &m->c[U->cells[i]];
            if (!cell_contains(m, c, rl, fsid, fsense)) continue;
            L->cell = U->cells[i];
            if (cell_near(m, c, rl, fsid)) *near |= F1;
            if (c->fill_kind == FILL_MAT) { o->daughter = -1; o->mc = c->mc; o->mat = c->fill; }
            else { o->daughter = c->fill; o->mc = -1; o->mat = -1;
                   for (int a = 0; a < 3; ++a) o->t[a] = c->tr[a]; }
            return 1;
        }
        return 0;
    }
    int idx;
    if (U->kind == U_RECT) {
        int ijk[3] = {0, 0, 0};
        int na = U->is2d ? 2 : 3;
        for (int a = 0; a < na; ++a) {
            ijk[a] = tile_index(U, a, rl[a]);
            if (fabs(rl[a] - tile_edge(U, a, ijk[a])) <= FLAG_DIST ||
                fabs(rl[a] - tile_edge(U, a, ijk[a] + 1)) <= FLAG_DIST) *near |= F1;
        }
        L->i = ijk[0]; L->j = ijk[1]; L->k = ijk[2];
        int in = 1;
        for (int a = 0; a < na; ++a) if (ijk[a] < 0 || ijk[a] >= U->n[a]) in = 0;
        idx = in ? ijk[0] + U->n[0] * (ijk[1] + U->n[1] * ijk[2]) : -1;
        for (int a = 0; a < 3; ++a)
            o->t[a] = (a < na) ? tile_centre(U, a, ijk[a]) : 0.0;
    } else {
        double t[3];
        hex_s(U, rl, t);
        int qc, rc;
        hex_cube_round(U, rl, &qc, &rc);
        /* brute force: every tile in a window around the guess; the owner must be unique */
        int nown = 0, qo = 0, ro = 0;
        for (int dq = -3; dq <= 3; ++dq)
            for (int dr = -3; dr <= 3; ++dr)
                if (hex_owns(U, qc + dq, rc + dr, t)) { nown++; qo = qc + dq; ro = rc + dr; }
        if (nown != 1) { qo = qc; ro = rc; *near |= F1; }
        double mm[3];
        hex_m(qo, ro, mm);
        for (int k = 0; k < 3; ++k)
            if (fabs(t[k] - U->pitch * (mm[k] - 0.5)) <= FLAG_DIST ||
                fabs(t[k] - U->pitch * (mm[k] + 0.5)) <= FLAG_DIST) *near |= F1;
        int kz = 0;
        if (U->nz > 0) {
            kz = rect_axis_index(U->zlo, U->zp, rl[2]);
            if (fabs(rl[2] - edge(U->zlo, U->zp, kz)) <= FLAG_DIST ||
                fabs(rl[2] - edge(U->zlo, U->zp, kz + 1)) <= FLAG_DIST) *near |= F1;
        }
        L->i = qo; L->j = ro; L->k = kz;
        int R = U->rings - 1, W = 2 * R + 1;
        int a = abs(qo), b = abs(ro), c = abs(qo + ro);
        int d = a > b ? a : b; d = d > c ? d : c;
        int in = d <= R && (U->nz == 0 || (kz >= 0 && kz < U->nz));
        idx = in ? U->hexmap[(ro + R) * W + (qo + R)] + (U->nz > 0 ? kz * (U->nfill / U->nz) : 0) : -1;
        o->t[0] = U->C[0] + ((double)qo * U->a1[0] + (double)ro * U->a2[0]);
        o->t[1] = U->C[1] + ((double)qo * U->a1[1] + (double)ro * U->a2[1]);
        o->t[2] = U->nz > 0 ? U->zlo + ((double)kz + 0.5) * U->zp : 0.0;
    }
    int d = idx >= 0 ? U->fill[idx] : U->outer;
    if (d < 0) return 0;                                       /* no outer: LOST */
    o->daughter = d; o->mc = -1; o->mat = -1;
    return 1;
}

/* Alg. 7 descent from level l0 (universe u, frame T) until a material cell */
static int descend(const Model *m, Level *S, int l0, int u, const double T[3], const double r[3],
                   int fsid, int fsense, int *depth, int *mc, int *mat, int *flags) {
    double Tc[3] = {T[0], T[1], T[2]};
    for (int l = l0; l < MAXD; ++l) {
        double rl[3];
        local_pos(r, Tc, rl);
        LocOut o;
        int near = 0;
        S[l].T[0] = Tc[0]; S[l].T[1] = Tc[1]; S[l].T[2] = Tc[2];
        if (!locate(m, u, rl, l == l0 ? fsid : -1, fsense, &S[l], &o, &near)) return 0;
        *flags |= near;
        if (o.daughter < 0) { *depth = l + 1; *mc = o.mc; *mat = o.mat; return 1; }
        Tc[0] = Tc[0] + o.t[0]; Tc[1] = Tc[1] + o.t[1]; Tc[2] = Tc[2] + o.t[2];
        u = o.daughter;
    }
    return 0;
}

/* ======================================================================
 * Distance to boundary over all levels (Table 1; O11, O13)
 * ====================================================================== */
typedef struct { double best, d2; int lstar, jstar; } Best;

static void consider(Best *b, double d, int l, int j) {
    if (d < b->best) { b->d2 = b->best; b->best = d; b->lstar = l; b->jstar = j; }
    else if (d < b->d2) b->d2 = d;
}

static void level_distances(const Model *m, const Level *L, int l, const double r[3], const double om[3],
                            int os_l, int os_s, Best *b, uint64_t *ev) {
    const Univ *U = &m->u[L->u];
    double rl[3];
    local_pos(r, L->T, rl);
    if (U->kind == U_CSG) {
        const Cell *c = &m->c[L->cell];
        for (int h = 0; h < c->n; ++h) {
            int sid = c->sid[h];
            double d = surf_dist(&m->s[sid], c->sense[h], os_l == l && os_s == sid, rl, om, ev);
            if (d < INFINITY) consider(b, d, l, sid);
        }
    } else if (U->kind == U_RECT) {
        int ijk[3] = {L->i, L->j, L->k};
        int na = U->is2d ? 2 : 3;
        for (int a = 0; a < na; ++a) {
            double u = om[a], d;
            const double e = u > 0.0 ? tile_edge(U, a, ijk[a] + 1) : tile_edge(U, a, ijk[a]);
            if (u == 0.0 || isinf(e)) continue;              /* no wall that way (N1 slabs) */
            d = (e - rl[a]) / u;
            if (ev) ev[E_RECT]++;
            consider(b, clamp0(d), l, 2 * a + (u > 0.0));
        }
    } else {
        double t[3], mm[3];
        hex_s(U, rl, t);
        hex_m(L->i, L->j, mm);
        if (ev) ev[E_HEX]++;
        for (int k = 0; k < 3; ++k) {
            double g = U->nrm[k][0] * om[0] + U->nrm[k][1] * om[1];
            if (g > 0.0) consider(b, clamp0((U->pitch * (mm[k] + 0.5) - t[k]) / g), l, k);
            else if (g < 0.0) consider(b, clamp0((U->pitch * (mm[k] - 0.5) - t[k]) / g), l, k + 3);
        }
        if (U->nz > 0) {
            double w = om[2];
            if (w > 0.0) consider(b, clamp0((edge(U->zlo, U->zp, L->k + 1) - rl[2]) / w), l, 7);
            else if (w < 0.0) consider(b, clamp0((edge(U->zlo, U->zp, L->k) - rl[2]) / w), l, 6);
        }
    }
}

/* ======================================================================
 * The walk (Alg. 2)
 * ====================================================================== */
typedef struct {
    uint64_t pid; double s; uint32_t seg; int32_t cell_before, cell_after, j;
    uint8_t kind; int8_t level; uint8_t terminal; uint8_t pad; uint32_t flags;
} TraceRec;   /* 40 bytes, layout documented in include/nestrack.h (nt_trace_rec) */

typedef struct { double sum, comp; } Neu;
static void neu_add(Neu *a, double x) {        /* Neumaier compensated summation */
    double t = a->sum + x;
    if (fabs(a->sum) >= fabs(x)) a->comp += (a->sum - t) + x;
    else a->comp += (x - t) + a->sum;
    a->sum = t;
}

typedef struct {
    Neu *len; uint64_t *exits; uint64_t cnt[NCOUNT]; uint64_t ev[NEVAL];
    Neu *mesh;                   /* per-voxel track length (M1), NULL when not tallied */
    Neu *inst;                   /* per-instance track length (D1), NULL when not tallied */
} Acc;

typedef struct {
    const Model *m; uint64_t seed, pid0, n, max_seg;
    double lo[3], w[3];
    const double *states;    /* optional explicit births: SoA 6 x n */
    uint8_t *pflags; TraceRec *trace; uint64_t trace_cap; uint64_t *trace_count;
    double *mesh_out;        /* optional per-voxel track length (M1), accumulated */
    double *inst_out;        /* optional per-instance track length (D1), accumulated */
    double *bank;            /* optional fission sites (F1): [n][max_sites][3] */
    uint8_t *bank_n;         /*   sites banked by each history */
    int max_sites;
    uint32_t *pnseg;         /* optional per-history segment count */
    uint8_t *pterm;          /* optional per-history terminal (T_*) */
} RunCtx;

static void emit(const RunCtx *R, uint64_t pid, uint32_t seg, int kind, int level, int j, int cb,
                 int ca, double s, int terminal, uint32_t flags) {
    if (!R->trace) return;
    uint64_t slot;
#pragma omp atomic capture
    slot = (*R->trace_count)++;
    if (slot >= R->trace_cap) return;
    TraceRec *t = &R->trace[slot];
    memset(t, 0, sizeof(*t));
    t->pid = pid; t->s = s; t->seg = seg; t->cell_before = cb; t->cell_after = ca; t->j = j;
    t->kind = (uint8_t)kind; t->level = (int8_t)level; t->terminal = (uint8_t)terminal; t->flags = flags;
}

/* D1: the instance index of the material cell reached by the stack S[0 .. depth-1]: the number
 * of instances that precede it in the enumeration, i.e. the leaves of every earlier sibling at
 * every level (earlier cells of the CSG universe, earlier tiles of the array; the outer universe
 * comes after every tile). */
static long instance_of(const Model *m, const Level *S, int depth) {
    long inst = 0;
    for (int l = 0; l < depth; ++l) {
        const Univ *U = &m->u[S[l].u];
        if (U->kind == U_CSG) {
            for (int i = 0; i < U->ncells && U->cells[i] != S[l].cell; ++i) {
                const Cell *c = &m->c[U->cells[i]];
                inst += c->fill_kind == FILL_MAT ? 1 : m->leaves[c->fill];
            }
        } else {
            int idx;
            if (U->kind == U_RECT) {
                int in = S[l].i >= 0 && S[l].i < U->n[0] && S[l].j >= 0 && S[l].j < U->n[1] &&
                         (U->is2d || (S[l].k >= 0 && S[l].k < U->n[2]));
                idx = in ? S[l].i + U->n[0] * (S[l].j + U->n[1] * (U->is2d ? 0 : S[l].k)) : U->nfill;
            } else {
                int R = U->rings - 1, W = 2 * R + 1, q = S[l].i, r = S[l].j, kz = S[l].k;
                int a = abs(q), b = abs(r), c = abs(q + r);
                int d = a > b ? a : b; d = d > c ? d : c;
                int in = d <= R && (U->nz == 0 || (kz >= 0 && kz < U->nz));
                idx = in ? U->hexmap[(r + R) * W + (q + R)] + (U->nz > 0 ? kz * (U->nfill / U->nz) : 0) : U->nfill;
            }
            for (int t = 0; t < idx; ++t) inst += m->leaves[U->fill[t]];
        }
    }
    return inst;
}

/* D1: the enumeration itself, by explicit depth-first recursion: out[i] = material-cell index of
 * instance i. */
static long enumerate_leaves(const Model *m, int u, int32_t *out, long pos) {
    const Univ *U = &m->u[u];
    if (U->kind == U_CSG) {
        for (int i = 0; i < U->ncells; ++i) {
            const Cell *c = &m->c[U->cells[i]];
            if (c->fill_kind == FILL_MAT) out[pos++] = c->mc;
            else pos = enumerate_leaves(m, c->fill, out, pos);
        }
    } else {
        for (int i = 0; i < U->nfill; ++i) pos = enumerate_leaves(m, U->fill[i], out, pos);
        if (U->outer >= 0) pos = enumerate_leaves(m, U->outer, out, pos);
    }
    return pos;
}

long orc_n_instances(void *vm) { Model *m = vm; return m->finalized ? m->leaves[m->root] : -1; }
long orc_instance_cells(void *vm, int32_t *out) {
    Model *m = vm;
    return m->finalized ? enumerate_leaves(m, m->root, out, 0) : -1;
}

/* M1: mesh plane i of axis a */
static double mesh_edge(const Model *m, int a, int i) { return m->mesh_lo[a] + (double)i * m->mesh_d[a]; }

/* M1: score the segment r + t om, t in [0, s], into the mesh: cut at every plane crossing,
 * sort the cuts, give each piece to the voxel holding its midpoint (plain definition). */
static void mesh_score(const Model *m, Acc *A, const double r[3], const double om[3], double s) {
    if (!A->mesh || !(s > 0.0)) return;
    int cap = 2 + m->mesh_n[0] + m->mesh_n[1] + m->mesh_n[2] + 3;
    double tl[2 + 4096];
    if (cap > 2 + 4096) return;                                  /* meshes here are <= 1024 / axis */
    int nt = 0;
    tl[nt++] = 0.0;
    tl[nt++] = s;
    for (int a = 0; a < 3; ++a) {
        if (om[a] == 0.0) continue;
        for (int i = 0; i <= m->mesh_n[a]; ++i) {
            double t = (mesh_edge(m, a, i) - r[a]) / om[a];
            if (t > 0.0 && t < s) tl[nt++] = t;
        }
    }
    /* insertion sort: the lists are short */
    for (int i = 1; i < nt; ++i) {
        double v = tl[i];
        int j = i - 1;
        while (j >= 0 && tl[j] > v) { tl[j + 1] = tl[j]; --j; }
        tl[j + 1] = v;
    }
    for (int k = 0; k + 1 < nt; ++k) {
        double t0 = tl[k], t1 = tl[k + 1];
        if (!(t1 > t0)) continue;
        double tm = (t0 + t1) * 0.5;
        int ijk[3], in = 1;
        for (int a = 0; a < 3 && in; ++a) {
            double x = r[a] + tm * om[a];
            int i = -1;
            for (int q = 0; q < m->mesh_n[a]; ++q)               /* explicit search: the definition */
                if (mesh_edge(m, a, q) <= x && x < mesh_edge(m, a, q + 1)) { i = q; break; }
            if (i < 0) in = 0;
            ijk[a] = i;
        }
        if (!in) continue;
        neu_add(&A->mesh[ijk[0] + m->mesh_n[0] * (ijk[1] + m->mesh_n[1] * ijk[2])], t1 - t0);
    }
}

int orc_set_mesh(void *vm, const double *lo, const double *hi, const int *n) {
    Model *m = vm;
    for (int a = 0; a < 3; ++a)
        if (n[a] < 1 || n[a] > 1024 || !(hi[a] > lo[a])) return -1;
    for (int a = 0; a < 3; ++a) {
        m->mesh_n[a] = n[a];
        m->mesh_lo[a] = lo[a];
        m->mesh_d[a] = (hi[a] - lo[a]) / (double)n[a];
    }
    m->mesh_on = 1;
    return 0;
}

static void walk(const RunCtx *R, uint64_t idx, Acc *A) {
    const Model *m = R->m;
    uint64_t pid = R->pid0 + idx;
    double r[3], om[3], tau;
    double xa, xb;
    /* W1 birth, epoch 0 (O17, O18) */
    draw(R->seed, pid, 0, 0, &xa, &xb);
    double xi_tau = xb;
    if (R->states) {
        for (int a = 0; a < 3; ++a) { r[a] = R->states[a * R->n + idx]; om[a] = R->states[(3 + a) * R->n + idx]; }
    } else {
        double xmu, xphi, xx, xy, xz, unused;
        draw(R->seed, pid, 0, 1, &xmu, &xphi);
        draw(R->seed, pid, 0, 2, &xx, &xy);
        draw(R->seed, pid, 0, 3, &xz, &unused);
        r[0] = R->lo[0] + R->w[0] * xx;
        r[1] = R->lo[1] + R->w[1] * xy;
        r[2] = R->lo[2] + R->w[2] * xz;
        iso(xmu, xphi, om);
    }
    tau = -orc_log(xi_tau);
    uint32_t epoch = 0, flags = 0;
    uint64_t nseg = 0;
    A->cnt[C_PARTICLES]++;

    Level S[MAXD];
    int depth = 0, mc = -1, mat = -1;
    int os_l = -1, os_s = -1;
    const double T0[3] = {0.0, 0.0, 0.0};
    int fl = 0;
    int terminal = T_NONE;
    if (!descend(m, S, 0, m->root, T0, r, -1, 0, &depth, &mc, &mat, &fl)) {
        flags |= (uint32_t)fl | F3;
        A->cnt[C_LOST]++;
        emit(R, pid, 0, EV_CROSS, -1, -1, -1, -1, 0.0, T_LOST, flags);
        terminal = T_LOST;
        goto done;
    }
    flags |= (uint32_t)fl;

    for (;;) {                                                    /* W2 */
        int cell = S[depth - 1].cell;
        const Mat *M = &m->m[mat];
        Best b = {INFINITY, INFINITY, -1, -1};
        for (int l = 0; l < depth; ++l) level_distances(m, &S[l], l, r, om, os_l, os_s, &b, A->ev);
        double ds = b.best;
        double dc = M->st > 0.0 ? tau / M->st : INFINITY;
        double g2 = b.d2 - ds, gc = fabs(dc - ds);
        if ((g2 > 0.0 && g2 <= FLAG_DIST) || (gc > 0.0 && gc <= FLAG_DIST)) flags |= F2;
        if (ds == INFINITY && dc == INFINITY) {                   /* nothing ahead: lost */
            flags |= F3; A->cnt[C_LOST]++;
            emit(R, pid, (uint32_t)nseg, EV_CROSS, -1, -1, cell, -1, 0.0, T_LOST, flags);
            terminal = T_LOST;
            goto done;
        }
        if (ds < dc) {                                            /* Alg. 2 "while d < tau/Sigma" */
            double s = ds;
            neu_add(&A->len[mc], s);
            mesh_score(m, A, r, om, s);
            if (A->inst) neu_add(&A->inst[instance_of(m, S, depth)], s);
            for (int a = 0; a < 3; ++a) r[a] = r[a] + s * om[a];
            double tt = tau - M->st * s;
            tau = tt > 0.0 ? tt : 0.0;                            /* O12 */
            nseg++;
            int l = b.lstar, j = b.jstar;
            if (l == 0 && m->u[S[0].u].kind == U_CSG && m->s[j].bc == BC_VACUUM) {
                A->exits[mc]++; A->cnt[C_CROSSINGS]++; A->cnt[C_LEAKS]++;
                emit(R, pid, (uint32_t)(nseg - 1), EV_LEAK, 0, j, cell, -1, s, T_LEAKED, flags);
                terminal = T_LEAKED;
                goto done;
            }
            if (l == 0 && m->u[S[0].u].kind == U_CSG && m->s[j].bc == BC_REFLECT) {
                om[m->s[j].kind] = -om[m->s[j].kind];            /* O19: PX/PY/PZ only */
                os_l = 0; os_s = j;
                A->cnt[C_REFLECTIONS]++;
                emit(R, pid, (uint32_t)(nseg - 1), EV_REFLECT, 0, j, cell, cell, s, T_NONE, flags);
            } else {
                A->exits[mc]++; A->cnt[C_CROSSINGS]++; A->cnt[C_CBL0 + l]++;
                const Univ *U = &m->u[S[l].u];
                int ok, fl2 = 0;
                if (U->kind == U_CSG) {                           /* O9': far side of j */
                    const Cell *oc = &m->c[S[l].cell];
                    int want = 0;
                    for (int h = 0; h < oc->n; ++h) if (oc->sid[h] == j) want = oc->sense[h] == POS ? NEG : POS;
                    ok = descend(m, S, l, S[l].u, S[l].T, r, j, want, &depth, &mc, &mat, &fl2);
                    os_l = l; os_s = j;
                } else {                                          /* Alg. 6: tile +- 1 */
                    Level *Lv = &S[l];
                    if (U->kind == U_RECT) {
                        int a = j / 2, dir = (j & 1) ? 1 : -1;
                        if (a == 0) Lv->i += dir; else if (a == 1) Lv->j += dir; else Lv->k += dir;
                    } else {
                        static const int dq[6] = {1, 0, -1, -1, 0, 1}, dr[6] = {0, 1, 1, 0, -1, -1};
                        if (j < 6) { Lv->i += dq[j]; Lv->j += dr[j]; }
                        else Lv->k += (j == 7) ? 1 : -1;
                    }
                    /* daughter of the new tile (fill or outer), tile-centred */
                    int idx, na, in = 1;
                    double t[3];
                    if (U->kind == U_RECT) {
                        int ijk[3] = {Lv->i, Lv->j, Lv->k};
                        na = U->is2d ? 2 : 3;
                        for (int a = 0; a < na; ++a) if (ijk[a] < 0 || ijk[a] >= U->n[a]) in = 0;
                        idx = in ? ijk[0] + U->n[0] * (ijk[1] + U->n[1] * ijk[2]) : -1;
                        for (int a = 0; a < 3; ++a)
                            t[a] = (a < na) ? tile_centre(U, a, ijk[a]) : 0.0;
                    } else {
                        int q = Lv->i, rr = Lv->j, kz = Lv->k;
                        int R = U->rings - 1, W = 2 * R + 1;
                        int aa = abs(q), bb = abs(rr), cc = abs(q + rr);
                        int dd = aa > bb ? aa : bb; dd = dd > cc ? dd : cc;
                        in = dd <= R && (U->nz == 0 || (kz >= 0 && kz < U->nz));
                        idx = in ? U->hexmap[(rr + R) * W + (q + R)] + (U->nz > 0 ? kz * (U->nfill / U->nz) : 0) : -1;
                        t[0] = U->C[0] + ((double)q * U->a1[0] + (double)rr * U->a2[0]);
                        t[1] = U->C[1] + ((double)q * U->a1[1] + (double)rr * U->a2[1]);
                        t[2] = U->nz > 0 ? U->zlo + ((double)kz + 0.5) * U->zp : 0.0;
                    }
                    int d = idx >= 0 ? U->fill[idx] : U->outer;
                    if (d < 0) ok = 0;
                    else {
                        double T1[3] = {Lv->T[0] + t[0], Lv->T[1] + t[1], Lv->T[2] + t[2]};
                        ok = descend(m, S, l + 1, d, T1, r, -1, 0, &depth, &mc, &mat, &fl2);
                    }
                    os_l = -1; os_s = -1;
                }
                flags |= (uint32_t)fl2;
                if (!ok) {
                    flags |= F3; A->cnt[C_LOST]++;
                    emit(R, pid, (uint32_t)(nseg - 1), EV_CROSS, l, j, cell, -1, s, T_LOST, flags);
                    terminal = T_LOST;
                    goto done;
                }
                emit(R, pid, (uint32_t)(nseg - 1), EV_CROSS, l, j, cell, S[depth - 1].cell, s, T_NONE, flags);
            }
        } else {                                                  /* collision at tau/Sigma */
            double s = dc;
            neu_add(&A->len[mc], s);
            mesh_score(m, A, r, om, s);
            if (A->inst) neu_add(&A->inst[instance_of(m, S, depth)], s);
            for (int a = 0; a < 3; ++a) r[a] = r[a] + s * om[a];
            nseg++;
            A->cnt[C_COLLISIONS]++;
            os_l = -1; os_s = -1;
            epoch++;
            draw(R->seed, pid, epoch, 0, &xa, &xb);
            if (xa < M->pabs) {                                   /* O14 absorption */
                A->cnt[C_ABSORPTIONS]++;
                if (R->bank && M->nut > 0.0) {                    /* F1: floor(nut + xi) sites here */
                    int ns = (int)floor(M->nut + xb);
                    if (ns > R->max_sites) ns = R->max_sites;     /* cannot happen: max_sites > nut */
                    for (int k = 0; k < ns; ++k)
                        for (int a = 0; a < 3; ++a) R->bank[((size_t)idx * R->max_sites + k) * 3 + a] = r[a];
                    R->bank_n[idx] = (uint8_t)ns;
                }
                emit(R, pid, (uint32_t)(nseg - 1), EV_COLLIDE, -1, -1, cell, cell, s, T_ABSORBED, flags);
                terminal = T_ABSORBED;
                goto done;
            }
            double xt = xb, xmu, xphi;
            draw(R->seed, pid, epoch, 1, &xmu, &xphi);
            iso(xmu, xphi, om);                                   /* O15 isotropic scatter */
            tau = -orc_log(xt);
            emit(R, pid, (uint32_t)(nseg - 1), EV_COLLIDE, -1, -1, cell, cell, s, T_NONE, flags);
        }
        if (nseg >= R->max_seg) {
            flags |= F3; A->cnt[C_CAPPED]++;
            terminal = T_CAPPED;
            emit(R, pid, (uint32_t)nseg, EV_COLLIDE, -1, -1, S[depth - 1].cell, -1, 0.0, terminal, flags);
            goto done;
        }
    }
done:
    A->cnt[C_SEGMENTS] += nseg;
    if (flags) A->cnt[C_FLAGGED]++;
    if (R->pflags) R->pflags[idx] = (uint8_t)flags;
    if (R->pnseg) R->pnseg[idx] = (uint32_t)nseg;
    if (R->pterm) R->pterm[idx] = (uint8_t)terminal;
}

static int run_common(void *vm, uint64_t seed, uint64_t pid0, uint64_t n, const double *lo,
                      const double *hi, const double *states, uint64_t max_seg, int nthreads,
                      double *out, uint8_t *pflags, void *trace, uint64_t trace_cap,
                      uint64_t *trace_count, uint64_t *evals, double *mesh_out, double *inst_out,
                      double *bank, uint8_t *bank_n, uint32_t *pnseg, uint8_t *pterm) {
    Model *m = vm;
    if (!m->finalized) return -1;
    RunCtx R;
    memset(&R, 0, sizeof(R));
    R.m = m; R.seed = seed; R.pid0 = pid0; R.n = n; R.max_seg = max_seg ? max_seg : 1000000;
    R.states = states; R.pflags = pflags; R.trace = trace; R.trace_cap = trace_cap;
    R.trace_count = trace_count;
    R.mesh_out = m->mesh_on ? mesh_out : NULL;
    R.inst_out = inst_out;
    R.bank = bank; R.bank_n = bank_n; R.max_sites = orc_max_sites(m);
    R.pnseg = pnseg; R.pterm = pterm;
    if (bank_n) memset(bank_n, 0, (size_t)n);
    const size_t ninst = inst_out ? (size_t)m->leaves[m->root] : 0;
    const size_t nbins = m->mesh_on ? (size_t)m->mesh_n[0] * m->mesh_n[1] * m->mesh_n[2] : 0;
    for (int a = 0; a < 3; ++a) { R.lo[a] = lo ? lo[a] : 0.0; R.w[a] = lo ? hi[a] - lo[a] : 0.0; }
    int nmc = m->n_mc;
    int T = nthreads > 0 ? nthreads : 1;
#ifndef _OPENMP
    T = 1;
#endif
    Acc *acc = calloc((size_t)T, sizeof(Acc));
    for (int t = 0; t < T; ++t) {
        acc[t].len = calloc((size_t)nmc + 1, sizeof(Neu));
        acc[t].exits = calloc((size_t)nmc + 1, sizeof(uint64_t));
        acc[t].mesh = R.mesh_out ? calloc(nbins, sizeof(Neu)) : NULL;
        acc[t].inst = R.inst_out ? calloc(ninst, sizeof(Neu)) : NULL;
    }
#pragma omp parallel num_threads(T)
    {
        int t = 0, nt = 1;
#ifdef _OPENMP
        t = omp_get_thread_num(); nt = omp_get_num_threads();
#endif
        uint64_t b = n * (uint64_t)t / (uint64_t)nt, e = n * (uint64_t)(t + 1) / (uint64_t)nt;
        for (uint64_t i = b; i < e; ++i) walk(&R, i, &acc[t]);   /* contiguous pid chunks */
    }
    /* merge in thread (= pid) order; accumulate into caller's out */
    for (int c = 0; c < nmc; ++c) {
        Neu tot = {0.0, 0.0};
        uint64_t ex = 0;
        for (int t = 0; t < T; ++t) { neu_add(&tot, acc[t].len[c].sum); neu_add(&tot, acc[t].len[c].comp); ex += acc[t].exits[c]; }
        out[c] += tot.sum + tot.comp;
        out[nmc + c] += (double)ex;
    }
    for (int k = 0; k < NCOUNT; ++k) {
        uint64_t v = 0;
        for (int t = 0; t < T; ++t) v += acc[t].cnt[k];
        out[2 * nmc + k] += (double)v;
    }
    if (evals)
        for (int k = 0; k < NEVAL; ++k) for (int t = 0; t < T; ++t) evals[k] += acc[t].ev[k];
    if (R.mesh_out)
        for (size_t v = 0; v < nbins; ++v) {
            Neu tot = {0.0, 0.0};
            for (int t = 0; t < T; ++t) { neu_add(&tot, acc[t].mesh[v].sum); neu_add(&tot, acc[t].mesh[v].comp); }
            R.mesh_out[v] += tot.sum + tot.comp;
        }
    if (R.inst_out)
        for (size_t v = 0; v < ninst; ++v) {
            Neu tot = {0.0, 0.0};
            for (int t = 0; t < T; ++t) { neu_add(&tot, acc[t].inst[v].sum); neu_add(&tot, acc[t].inst[v].comp); }
            R.inst_out[v] += tot.sum + tot.comp;
        }
    for (int t = 0; t < T; ++t) { free(acc[t].len); free(acc[t].exits); free(acc[t].mesh); free(acc[t].inst); }
    free(acc);
    return 0;
}

int orc_run(void *vm, uint64_t seed, uint64_t pid0, uint64_t n, const double *lo, const double *hi,
            uint64_t max_seg, int nthreads, double *out, uint8_t *pflags, void *trace,
            uint64_t trace_cap, uint64_t *trace_count, uint64_t *evals, double *mesh_out,
            double *inst_out, double *bank, uint8_t *bank_n, uint32_t *pnseg, uint8_t *pterm) {
    return run_common(vm, seed, pid0, n, lo, hi, NULL, max_seg, nthreads, out, pflags, trace,
                      trace_cap, trace_count, evals, mesh_out, inst_out, bank, bank_n, pnseg, pterm);
}

int orc_run_states(void *vm, uint64_t seed, uint64_t pid0, uint64_t n, const double *states,
                   uint64_t max_seg, int nthreads, double *out, uint8_t *pflags, void *trace,
                   uint64_t trace_cap, uint64_t *trace_count, uint64_t *evals, double *mesh_out,
                   double *inst_out, double *bank, uint8_t *bank_n, uint32_t *pnseg, uint8_t *pterm) {
    return run_common(vm, seed, pid0, n, NULL, NULL, states, max_seg, nthreads, out, pflags, trace,
                      trace_cap, trace_count, evals, mesh_out, inst_out, bank, bank_n, pnseg, pterm);
}

/* F1: source particles J = j_begin .. j_begin + n_next - 1 drawn from a flat site list (the
 * multi-rank form: the list is every rank's bank in rank, history, site order). */
void orc_source_from_sites(const double *sites, uint64_t M, uint64_t seed, uint32_t cycle, uint64_t j_begin,
                           uint64_t n_next, double *states_out) {
    for (uint64_t j = 0; j < n_next; ++j) {
        const uint64_t J = j_begin + j;
        double u, unused, xmu, xphi, om[3];
        draw(seed, J, cycle, 0xF155u, &u, &unused);
        const uint64_t t = (uint64_t)floor(u * (double)M);
        draw(seed, J, cycle, 0xF156u, &xmu, &xphi);
        iso(xmu, xphi, om);
        for (int a = 0; a < 3; ++a) {
            states_out[a * n_next + j] = sites[t * 3 + a];
            states_out[(3 + a) * n_next + j] = om[a];
        }
    }
}

/* F1: next-cycle source.  M = total banked sites (history order, then site order).  Source
 * particle j takes the site with flat index floor(u_j * M), u_j = first uniform of Philox block
 * (seed; j, cycle, 0xF155), and an isotropic direction from block (seed; j, cycle, 0xF156).
 * states_out: SoA [6][n_next].  Returns M (0: nothing banked, states untouched). */
uint64_t orc_fission_source(void *vm, const double *bank, const uint8_t *bank_n, uint64_t n_prev,
                            uint64_t seed, uint32_t cycle, uint64_t n_next, double *states_out) {
    Model *m = vm;
    const int ms = orc_max_sites(m);
    uint64_t M = 0;
    for (uint64_t h = 0; h < n_prev; ++h) M += bank_n[h];
    if (M == 0) return 0;
    for (uint64_t j = 0; j < n_next; ++j) {
        double u, unused, xmu, xphi, om[3];
        draw(seed, j, cycle, 0xF155u, &u, &unused);
        uint64_t t = (uint64_t)floor(u * (double)M);
        uint64_t h = 0, acc = 0;
        while (!(t < acc + bank_n[h])) { acc += bank_n[h]; ++h; }  /* the site's history (plain scan) */
        const double *site = bank + ((size_t)h * ms + (t - acc)) * 3;
        draw(seed, j, cycle, 0xF156u, &xmu, &xphi);
        iso(xmu, xphi, om);
        for (int a = 0; a < 3; ++a) {
            states_out[a * n_next + j] = site[a];
            states_out[(3 + a) * n_next + j] = om[a];
        }
    }
    return M;
}

/* ---------------------------------------------------------------- unit queries */

/* Alg. 7 point location for n points (xyz SoA 3 x n): material cell id (global) or -1 */
int orc_find_cells(void *vm, const double *xyz, uint64_t n, int32_t *cell_out, uint8_t *flag_out) {
    Model *m = vm;
    if (!m->finalized) return -1;
    for (uint64_t i = 0; i < n; ++i) {
        double r[3] = {xyz[i], xyz[n + i], xyz[2 * n + i]};
        Level S[MAXD];
        int depth, mc, mat, fl = 0;
        const double T0[3] = {0.0, 0.0, 0.0};
        int ok = descend(m, S, 0, m->root, T0, r, -1, 0, &depth, &mc, &mat, &fl);
        cell_out[i] = ok ? S[depth - 1].cell : -1;
        if (flag_out) flag_out[i] = (uint8_t)(fl | (ok ? 0 : F3));
    }
    return 0;
}

/* P16: number of cells of CSG universe uid containing the local point */
int orc_count_containing(void *vm, int uid, const double *r) {
    Model *m = vm;
    const Univ *U = &m->u[uid];
    int cnt = 0;
    for (int i = 0; i < U->ncells; ++i) cnt += cell_contains(m, &m->c[U->cells[i]], r, -1, 0);
    return cnt;
}

/* unit: distance to leave half-space (sid, sense) from r along om (O11) */
double orc_surface_distance(void *vm, int sid, int sense_pos, int onsurf, const double *r, const double *om) {
    Model *m = vm;
    return surf_dist(&m->s[sid], sense_pos ? POS : NEG, onsurf, r, om, NULL);
}

double orc_surface_f(void *vm, int sid, const double *r) { return surf_f(&((Model *)vm)->s[sid], r); }

/* unit: locate a local point in one array universe -> (i,j,k) or (q,r,kz), daughter, centre */
int orc_locate_array(void *vm, int uid, const double *rl, int32_t *ijk, int32_t *daughter, double *t,
                     int32_t *flag) {
    Model *m = vm;
    Level L;
    LocOut o;
    int near = 0;
    memset(&o, 0, sizeof(o));
    int ok = locate(m, uid, rl, -1, 0, &L, &o, &near);
    ijk[0] = L.i; ijk[1] = L.j; ijk[2] = L.k;
    *daughter = ok ? o.daughter : -1;
    for (int a = 0; a < 3; ++a) t[a] = o.t[a];
    *flag = near;
    return ok;
}

/* unit: hex ownership test in s-space for tile (q, r) */
int orc_hex_owns(void *vm, int uid, int q, int r, const double *rl) {
    Model *m = vm;
    double t[3];
    hex_s(&m->u[uid], rl, t);
    return hex_owns(&m->u[uid], q, r, t);
}

/* O15 direction of a scatter / birth draw pair, exposed for its statistical pins */
void orc_iso(double xmu, double xphi, double *om) { iso(xmu, xphi, om); }

int orc_ncount(void) { return NCOUNT; }
int orc_trace_rec_size(void) { return (int)sizeof(TraceRec); }

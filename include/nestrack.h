/* nestrack.h — C ABI of the B200-native nested-geometry tracking library
 * (libnestrack.so, built from paper_2406_13849_b200/csrc).
 *
 * The calls follow the paper's statement of the problem (arXiv 2406.13849,
 * PAPER.md): build a CSG model from surface primitives and Boolean cell
 * logic (§1, Fig. 2), universes and rect/hex arrays (P:133-145,
 * Fig. 3), accelerate CSG universes with a bounding interval hierarchy
 * (§4.3); then track a batch of particle histories with the
 * Table-1 operations (find_cell, distance_to_surface, move_within_cell,
 * cross_surface, change_direction) inside the random walk of
 * Alg. 2, scoring per-cell track length and crossing counts.
 * Numerical readings the paper leaves open are listed in DESIGN.md.
 *
 * ---- conventions -------------------------------------------------------
 * - Every call returns nt_status (NT_OK = 0, < 0 = error).  nt_last_error()
 *   returns a thread-local, library-owned, NUL-terminated message for the
 *   last failing call on the calling thread.  No C++ exception crosses the ABI.
 * - Ids are dense int32 in creation order: surfaces, materials, cells
 *   (global over all CSG universes), universes (CSG, rect and hex share one
 *   id space).  Forward references (a fill naming a universe created later)
 *   are allowed and validated by nt_finalize.
 * - The model (host tables and the device copy) is owned by the library.  It
 *   is immutable after nt_finalize; tracking calls may run concurrently on
 *   different streams (each call uses its own work counter slot, up to 64 in
 *   flight per model).
 * - Output buffers are CALLER-OWNED DEVICE memory on the finalize device
 *   (e.g. torch tensors).  nt_track* ACCUMULATE into `out` (zero it first).
 * - Calls that take `cuda_stream` (a cudaStream_t, NULL = legacy default
 *   stream) are asynchronous on that stream; asynchronous CUDA faults surface
 *   as NT_E_CUDA at the next call or at stream synchronisation.
 * - Lost and capped histories are counters, not errors.
 */
#ifndef NESTRACK_H
#define NESTRACK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NT_ABI_VERSION 4

typedef enum {
    NT_OK = 0,
    NT_E_ARG = -1,          /* bad pointer / size / enum value                          */
    NT_E_ID = -2,           /* id out of range                                          */
    NT_E_ORDER = -3,        /* builder call after finalize, or track before finalize    */
    NT_E_GEOMETRY = -4,     /* invalid model (see nt_finalize)                          */
    NT_E_UNSUPPORTED = -5,  /* e.g. NT_TRACKER_RECT on a model that is not rect-shaped  */
    NT_E_CUDA = -6,         /* CUDA runtime error (message has the CUDA error string)   */
    NT_E_NOMEM = -7         /* host or device allocation failed                         */
} nt_status;

/* Surface primitives: implicit function f, positive side f >= 0.
 *   NT_PX/PY/PZ coef {a}            : f = x - a  (resp. y, z)
 *   NT_PLANE    coef {nx,ny,nz,d}   : f = (nx x + ny y) + nz z - d   (not normalised)
 *   NT_CZ       coef {x0,y0,R}      : f = (dx dx + dy dy) - R R      (infinite cylinder along z)
 *   NT_SPHERE   coef {x0,y0,z0,R}   : f = ((dx dx + dy dy) + dz dz) - R R                   */
typedef enum { NT_PX = 0, NT_PY = 1, NT_PZ = 2, NT_PLANE = 3, NT_CZ = 4, NT_SPHERE = 5 } nt_surface_kind;

/* Boundary conditions, meaningful only on surfaces of root-universe cells.
 * VACUUM: the particle leaks.  REFLECT (PX/PY/PZ only): specular, one direction
 * component changes sign. */
typedef enum { NT_BC_NONE = 0, NT_BC_VACUUM = 1, NT_BC_REFLECT = 2 } nt_bc;
typedef enum { NT_FILL_MATERIAL = 0, NT_FILL_UNIVERSE = 1 } nt_fill_kind;
typedef enum { NT_HEX_POINTY = 0, NT_HEX_FLAT = 1 } nt_hex_orient;
/* GENERIC: any nesting of CSG (BIH), rect and hex universes.  RECT: the
 * rect-specialised comparison tracker of §3.3 (Alg. 9-10).  The rect tracker runs on
 * the ring event queues by default (the generic tracker's default scheduler, so the two compare
 * like for like) or history-based with NT_HISTORY; NT_WARPQ / NT_ROUNDS / NT_DP with it: NT_E_ARG. */
typedef enum { NT_TRACKER_GENERIC = 0, NT_TRACKER_RECT = 1 } nt_tracker;

/* nt_run.flags */
#define NT_TRACE 1u          /* write one nt_trace_rec per segment into outputs.trace */
/* Scheduler of the generic tracker (results are identical; only speed differs).  Default: event
 * queues per block (§2.3 event-based execution): a block owns block_dim particle slots
 * and alternates a MOVE stage and an EVENT stage (collide / descend / birth), each over queues
 * compacted with warp ballots, so every warp runs one event type on 32 slots at a time.         */
#define NT_HISTORY 2u        /* history-based persistent kernel: one history per thread            */
#define NT_WARPQ 4u          /* event queues per warp (64 slots per warp, no block barriers)      */
/* Dispatch of the tracking operations inside the block-queue scheduler (§4 methods):
 * default SP (switch on the universe kind).  NT_DP: dynamic polymorphism, every
 * find_cell / distance_to_boundary / array cross_surface is a virtual call on a per-universe
 * tracker object built on the device; results are identical.  Needs the generic
 * tracker, block queues (not NT_HISTORY / NT_WARPQ) and block_dim 0 or 256, else NT_E_ARG.
 * ST (pseudo-array universes) is the build option nt_build_opts.pseudo_array.   */
#define NT_DP 8u
/* Block queues run without rounds or block barriers by default: each event queue is a ring in
 * shared memory, a warp claims up to 32 entries of the fullest ring, runs that event and the move,
 * and appends each slot to the ring of its next event.  NT_ROUNDS selects the earlier round-based
 * form instead (every warp takes one 32-slot chunk per round, one block barrier per round); runs
 * with block_dim 128 always use rounds.  Results are identical.                                */
#define NT_ROUNDS 16u

/* Per-particle flag bits written to outputs.pflags (reading O16):
 *   F1: a cell/tile chosen by a descent has another surface within 1e-10 cm
 *   F2: a runner-up distance (or the collision distance) lies within 1e-10 cm above the chosen one
 *   F3: the history was LOST or CAPPED                                                    */
#define NT_F1 1u
#define NT_F2 2u
#define NT_F3 4u

/* Counter block at the end of the packed output (all exact integers stored as fp64). */
enum {
    NT_C_PARTICLES = 0, NT_C_SEGMENTS, NT_C_CROSSINGS, NT_C_REFLECTIONS, NT_C_LEAKS,
    NT_C_COLLISIONS, NT_C_ABSORPTIONS, NT_C_LOST, NT_C_CAPPED, NT_C_FLAGGED,
    NT_C_CROSS_LEVEL0,                 /* + level, 8 entries: crossings by surf_universe level */
    NT_NC = NT_C_CROSS_LEVEL0 + 8
};

/* Trace record kinds / terminals */
enum { NT_EV_CROSS = 0, NT_EV_REFLECT = 1, NT_EV_LEAK = 2, NT_EV_COLLIDE = 3 };
enum { NT_T_NONE = 0, NT_T_ABSORBED = 1, NT_T_LEAKED = 2, NT_T_LOST = 3, NT_T_CAPPED = 4 };

/* One segment of one history (40 bytes, little-endian, no padding beyond `pad`).
 *   pid, seg (0-based segment index), s = segment length (cm),
 *   cell_before / cell_after: global material-cell ids (-1 = none: leaked / lost),
 *   j = crossed surface id (CSG level), wall code 2*axis+(dir>0) (rect level),
 *       face 0..5 / 6 = z-, 7 = z+ (hex level), -1 for collisions,
 *   level = surf_universe level of the crossing (-1 for collisions),
 *   terminal = NT_T_*, flags = the particle's O16 bits so far.
 * A history lost at birth writes one record (seg 0, level -1, terminal LOST);
 * a capped history writes an extra record (seg = nseg, terminal CAPPED). */
typedef struct {
    uint64_t pid;
    double s;
    uint32_t seg;
    int32_t cell_before, cell_after, j;
    uint8_t kind;
    int8_t level;
    uint8_t terminal;
    uint8_t pad;
    uint32_t flags;
} nt_trace_rec;

typedef struct nt_model nt_model;

/* ---- errors / version ---------------------------------------------------- */
const char* nt_last_error(void);
int32_t nt_abi_version(void);

/* ---- model building (host only) --------------------------------- */
nt_status nt_model_create(nt_model** out);
void nt_model_destroy(nt_model* m);                  /* frees host and device copies; NULL ok */

/* coef: 1 (PX/PY/PZ), 4 (PLANE), 3 (CZ), 4 (SPHERE) doubles, copied. */
nt_status nt_add_surface(nt_model* m, nt_surface_kind kind, const double* coef, nt_bc bc, int32_t* id);

/* One-group macroscopic cross sections (1/cm): 0 <= sigma_a <= sigma_t (sigma_t = 0: void). */
nt_status nt_add_material(nt_model* m, double sigma_t, double sigma_a, int32_t* id);

/* One-group fission (Alg. 1-2; reading F1): material
 * `mat` gets nu*Sigma_f >= 0 (> 0 needs sigma_a > 0; nu_sigma_f / sigma_a <= 200).  An absorption
 * in it then banks floor(nu_sigma_f / sigma_a + xi) fission sites at the absorption point when
 * the run passes outputs.bank.  NT_E_ID for a bad id; values are validated at nt_finalize. */
nt_status nt_set_fission(nt_model* m, int32_t mat, double nu_sigma_f);

nt_status nt_add_csg_universe(nt_model* m, int32_t* uid);

/* A cell of CSG universe `uid` = intersection of signed half-spaces (Fig. 2):
 * halfspaces[i] = +(surf+1) for the positive side, -(surf+1) for the negative side;
 * n = 0 means all space.  fill = material id (NT_FILL_MATERIAL) or daughter universe id
 * (NT_FILL_UNIVERSE) placed with `translation` (NULL = 0; daughter frame = parent - t). */
nt_status nt_add_cell(nt_model* m, int32_t uid, const int32_t* halfspaces, int32_t n,
                      nt_fill_kind fill_kind, int32_t fill, const double translation[3],
                      int32_t* cell_id);

/* Uniform rectilinear array universe (Fig. 3; Alg. 5-6).  Tile (i,j,k) spans
 * [ll + i p, ll + (i+1) p) per axis; pitch[2] == 0 makes a 2-D array (shape[2] ignored,
 * infinite in z).  fill: shape[0]*shape[1]*shape[2] universe ids, x fastest.  Tiles
 * outside the shape take `outer_uid` (-1 = none: a particle reaching one is LOST).
 * Daughters are placed at the tile centre. */
nt_status nt_add_rect_array(nt_model* m, const double lower_left[3], const double pitch[3],
                            const int32_t shape[3], const int32_t* fill, int32_t outer_uid,
                            int32_t* uid);

/* Non-uniform rectilinear array (Alg. 5 find_cell by binary search over the mesh divisions,
 * P:513-525; non-uniform spacing for inter-assembly gaps; reading N1).
 * edges: n_edges[0] x divisions, then n_edges[1] y, then n_edges[2] z, each strictly
 * increasing and finite (copied); n_edges[2] == 0 makes the array 2-D (infinite in z).  Tile
 * (i, j, k) spans [e_i, e_i+1) per axis; points below the first / at or above the last division
 * lie in the outer slabs (index -1 / n), which take `outer_uid`.  Daughters are placed at the
 * tile centre (e_i + e_i+1) * 0.5 (slabs: at the division they touch).  fill: x fastest.
 * NT_E_GEOMETRY for fewer than 2 edges on an axis or non-increasing edges (at nt_finalize).
 * Not rect-specialisable (NT_TRACKER_RECT rejects the model). */
nt_status nt_add_rect_edges(nt_model* m, const double* edges, const int32_t n_edges[3],
                            const int32_t* fill, int32_t outer_uid, int32_t* uid);

/* Hexagonal array universe (Fig. 3; indexing omitted by the paper, P:444-448 — DESIGN.md
 * reading O9).  Axial (q, r), pitch = flat-to-flat distance, rings >= 1 (1 + 3 rings(rings-1)
 * tiles).  fill order: r ascending, then q ascending over max(|q|,|r|,|q+r|) <= rings-1;
 * with z_pitch > 0 the pattern repeats for nz layers from z_lower (z slowest). */
nt_status nt_add_hex_array(nt_model* m, nt_hex_orient orient, const double center[2], double pitch,
                           int32_t rings, double z_lower, double z_pitch, int32_t nz,
                           const int32_t* fill, int32_t outer_uid, int32_t* uid);

nt_status nt_set_root(nt_model* m, int32_t uid);

/* Superimposed Cartesian mesh track-length tally (the paper's active-cycle
 * 119x119x30 mesh tally; reading M1).  Voxel (i, j, k) spans
 * [lo_a + i d_a, lo_a + (i+1) d_a) per axis with d_a = (hi_a - lo_a) / shape_a (global frame).
 * When a run passes nt_outputs.mesh, every segment adds to each voxel the length of its part
 * inside that voxel (parts outside the mesh are not scored).  1 <= shape_a <= 4096, hi > lo,
 * else NT_E_GEOMETRY.  Call before nt_finalize; a later call replaces the mesh. */
nt_status nt_set_mesh(nt_model* m, const double lo[3], const double hi[3], const int32_t shape[3]);

/* ---- finalize: validate, BIH (SAH), optional pseudo-arrays, flatten, upload -------- */
typedef struct {
    int32_t device;         /* CUDA device for the geometry copy; -1 = host-only build (no upload) */
    int32_t bih_max_leaf;   /* max cells per BIH leaf (default 4)                                 */
    int32_t pseudo_array;   /* 1: convert rect/hex arrays to CSG "pseudo-array" universes (§4.3 ST) */
    int32_t reserved;
    double sah_ct, sah_ci;  /* SAH traversal / intersection cost weights (default 1, 1)           */
} nt_build_opts;

void nt_build_opts_default(nt_build_opts* o);

/* Errors: NT_E_GEOMETRY for an invalid model: bad surface reference or duplicate surface in a
 * cell, cylinder/sphere R <= 0, zero plane normal, REFLECT on a non-axis plane, a BC-tagged
 * surface referenced outside the root universe, bad array parameters, a universe cycle,
 * nesting depth > 8, a material with sigma_a > sigma_t or negative cross sections.
 * NT_E_ORDER if already finalized.  NT_E_CUDA / NT_E_NOMEM on upload failure. */
nt_status nt_finalize(nt_model* m, const nt_build_opts* opts);

typedef struct {
    int32_t n_surfaces, n_cells, n_material_cells, n_universes, max_depth;
    int32_t rect_specialisable;   /* 1 if NT_TRACKER_RECT accepts the model */
    int32_t rect_levels;          /* number of rect array levels the rect tracker unrolls */
    int32_t n_bih_nodes;
    int64_t out_len;              /* 2*n_material_cells + NT_NC */
    size_t device_bytes;          /* size of the device geometry blob */
    int64_t mesh_bins;            /* voxels of the mesh set by nt_set_mesh (0: none) */
    int64_t n_instances;          /* material-cell instances (reading D1); 0 for pseudo-array
                                     builds or more than 2^31 - 1 instances (no instance tallies) */
    int32_t max_sites;            /* fission sites one absorption can bank: floor(max nu_sigma_f/sigma_a) + 1 */
} nt_model_info;

nt_status nt_model_info_get(const nt_model* m, nt_model_info* info);

/* Next cycle's fission source (F1, Alg. 1 power iteration): from the bank of n_prev histories
 * (outputs.bank / bank_n of the previous nt_track*), draw n_next birth states into d_states
 * (device SoA fp64 [6][n_next], for nt_track_states): particle j takes the site with flat index
 * floor(u_j * M) in (history, site) order, M = total sites, u_j the first uniform of Philox block
 * (key seed; counter j, cycle, 0xF155), and an isotropic direction from block (j, cycle, 0xF156).
 * *total_sites = M; M = 0 leaves d_states untouched (the caller decides: subcritical collapse).
 * Synchronises `cuda_stream` (M is needed on the host). */
nt_status nt_fission_source(nt_model* m, const double* d_bank, const uint8_t* d_bank_n, uint64_t n_prev,
                            uint64_t seed, uint32_t cycle, uint64_t n_next, double* d_states,
                            uint64_t* total_sites, void* cuda_stream);

/* The two halves of nt_fission_source, for multi-GPU power iteration (the all-gather of the sites
 * happens between them, see paper_2406_13849_b200.power_iteration_distributed):
 * nt_bank_compact writes the banked sites as a flat list in (history, site) order into d_sites
 * (device, capacity n * max_sites * 3 fp64) and returns their number (synchronises the stream);
 * nt_source_from_sites draws source particles J = j_begin .. j_begin + n_next - 1 from a flat list
 * of total_sites sites (site floor(u_J * total_sites), u_J from Philox(seed; J, cycle, 0xF155),
 * direction from block 0xF156) into d_states [6][n_next].  NT_E_ARG when total_sites = 0. */
nt_status nt_bank_compact(nt_model* m, const double* d_bank, const uint8_t* d_bank_n, uint64_t n, double* d_sites,
                          uint64_t* total_sites, void* cuda_stream);
nt_status nt_source_from_sites(nt_model* m, const double* d_sites, uint64_t total_sites, uint64_t seed,
                               uint32_t cycle, uint64_t j_begin, uint64_t n_next, double* d_states,
                               void* cuda_stream);

/* Per-instance tallies (reading D1): material-cell instances are numbered by a depth-first
 * enumeration of the model -- a CSG universe's cells in id order (a material cell is one
 * instance, a fill cell contributes its universe's instances), an array's tiles in fill order,
 * then its outer universe once.  out[i] = material-cell bin of instance i; writes
 * min(cap, n_instances) entries.  NT_E_ORDER before nt_finalize. */
nt_status nt_instance_cells(const nt_model* m, int32_t* out, int64_t cap);

/* Tally bin b (0 <= b < n_material_cells) -> global cell id, ascending; writes min(cap, n). */
nt_status nt_material_cell_ids(const nt_model* m, int32_t* out, int32_t cap);

/* BIH introspection of CSG universe uid (tests): node count, depth, and the cells of all
 * leaves in leaf order (each cell exactly once). */
nt_status nt_bih_info(const nt_model* m, int32_t uid, int32_t* n_nodes, int32_t* depth,
                      int32_t* leaf_cells, int32_t cap, int32_t* n_leaf_cells);

/* ---- tracking (Alg. 2; event handling DESIGN.md) -------------------------- */
typedef struct {
    uint64_t seed;            /* Philox key (reading O17)                                     */
    uint64_t pid_begin, n;    /* histories pid_begin .. pid_begin+n-1                         */
    double src_lo[3], src_hi[3]; /* uniform source box (O18); unused by nt_track_states      */
    uint64_t max_segments;    /* per history; 0 = 1e6; reaching it -> CAPPED                  */
    int32_t tracker;          /* nt_tracker                                                   */
    uint32_t flags;           /* NT_TRACE                                                     */
    int32_t block_dim;        /* 0 = auto (256); block queues: 128 or 256; ignored by NT_WARPQ */
    int32_t blocks_per_sm;    /* 0 = auto (tuning knob)                                       */
} nt_run;

typedef struct {
    double* out;              /* device, out_len fp64: [len(n_mc) | exits(n_mc) | counters(NT_NC)], accumulated */
    uint8_t* pflags;          /* device, optional (NULL), n entries: O16 bits per history     */
    uint32_t* pnseg;          /* device, optional (NULL), n entries: segments of each history */
    uint8_t* pterm;           /* device, optional (NULL), n entries: NT_T_* terminal of each history */
    nt_trace_rec* trace;      /* device, optional: records in arbitrary order                  */
    uint64_t trace_cap;       /* capacity of trace in records                                  */
    uint64_t* trace_count;    /* device, required with NT_TRACE: records attempted (may exceed cap) */
    double* mesh;             /* device, optional (NULL = no mesh tally): per-voxel track length of the
                                 model's mesh (nt_set_mesh), x fastest, accumulated; ignored when the
                                 model has no mesh */
    double* inst;             /* device, optional (NULL = none): track length per material-cell instance
                                 (distributed-cell tally, reading D1), n_instances entries,
                                 accumulated.  Generic tracker, no NT_TRACE, no pseudo-array build,
                                 else NT_E_UNSUPPORTED */
    double* bank;             /* device, optional (NULL = no fission bank, F1): n * max_sites * 3 fp64,
                                 site k of history i at [(i * max_sites + k) * 3] (x, y, z) */
    uint8_t* bank_n;          /* device, with bank: n entries, sites banked by each history (zeroed
                                 by the call first); k = sum(bank_n) / n is the cycle's estimate */
} nt_outputs;

/* Track run->n histories born from (seed, pid) in the source box. Asynchronous on cuda_stream. */
nt_status nt_track(nt_model* m, const nt_run* run, const nt_outputs* o, void* cuda_stream);

/* Same walk with explicit birth states: d_states = device SoA fp64 [6][n] = x,y,z,u,v,w
 * (direction need not be re-normalised); tau is still drawn from (seed, pid). */
nt_status nt_track_states(nt_model* m, const nt_run* run, const double* d_states,
                          const nt_outputs* o, void* cuda_stream);

/* End-to-end host entry point: HOST output buffer (out_len fp64, overwritten), device
 * scratch owned by the library; copies in/out and synchronises cuda_stream. */
nt_status nt_track_host(nt_model* m, const nt_run* run, double* host_out, void* cuda_stream);

/* Point location (Alg. 7) for n points: d_xyz = device SoA fp64 [3][n];
 * d_cell[i] = global material-cell id or -1 (lost); d_flag (optional) = O16 bits. */
nt_status nt_find_cells(nt_model* m, const double* d_xyz, uint64_t n, int32_t* d_cell,
                        uint8_t* d_flag, void* cuda_stream);

/* Number of kernel launches issued by the last tracking call on this model (evidence). */
int32_t nt_last_launch_count(const nt_model* m);

/* Device self-test of the kernels' fp64 division / square root (nt_math.cuh fdiv, fsqrt) against
 * the IEEE `/` and sqrt on n random operand pairs spanning the walk's ranges.
 * mismatches[0] = division mismatches, mismatches[1] = sqrt mismatches (host array of 2).
 * Synchronous on the current device. */
nt_status nt_selftest_arith(uint64_t n, uint64_t seed, uint64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif /* NESTRACK_H */

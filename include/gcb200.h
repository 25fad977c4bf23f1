/*
 * gcb200.h - C-ABI of the B200-native GCA-H2 hot path (libgcb200.so).
 *
 * Plain C: pointers, sizes and an opaque cudaStream_t passed as void*.
 * Every pointer marked [dev] is caller-owned device memory (the Python host
 * layer allocates it with torch); [host] pointers are host memory.  All
 * functions are thread-safe (no global mutable state besides the error
 * string, which is thread-local, and an atomic launch counter) and never
 * synchronise the device unless stated.  Return value: GC_OK or one of the
 * GC_ERR_* codes; gc_last_error() returns the message.  The host layer maps
 * GC_ERR_CONFIG -> ConfigError, GC_ERR_GEOMETRY -> GeometryError,
 * GC_ERR_STATE -> StateError and everything else -> GreencrossError
 * (greencross/errors.py:4-35).
 *
 * Each entry point names the reference interface whose results it
 * reproduces (paths relative to /root/reference/pkg/src/greencross).
 */
#ifndef GCB200_H
#define GCB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_ABI_VERSION 3

#define GC_OK 0
#define GC_ERR_CONFIG 1
#define GC_ERR_GEOMETRY 2
#define GC_ERR_CUDA 3
#define GC_ERR_STATE 4

int gc_abi_version(void);
const char* gc_last_error(void);
/* kernels launched by this library since load / last reset (bench evidence) */
uint64_t gc_launch_count(void);
void gc_reset_launch_count(void);

/* ---------------------------------------------------------------------
 * Device-resident geometry (replaces geometry.chart_pack, geometry.py:266-293,
 * and assembly._surface_quadrature, assembly.py:371-381).
 *   corners [dev] (nt,3,3)  triangle vertices
 *   gram    [dev] (nt,)     plane Gramian |(v1-v0)x(v2-v0)| from the host
 *   tri_vid [dev] (nt,3)    global vertex ids (pair classification)
 *   xq      [dev] (nt,mq,3) regular-rule surface points (gc_surface_points)
 *   wq      [dev] (mq,)     triangle_gauss(q_reg) weights
 *   wq_host [host] (mq,)    the same weights (kernel-parameter copies)
 * ------------------------------------------------------------------- */
typedef struct gc_geom {
    const double* corners;
    const double* gram;
    const int64_t* tri_vid;
    const double* xq;
    const double* wq;
    int64_t nt;
    int64_t mq;
    const double* wq_host;
    /* [dev] nt x 3 chart normal of each plane triangle, |n| = gram
     * (geometry.py:281-290); read by the double-layer kernel only */
    const double* normals;
    /* 0 = single layer 1/(4 pi r), 1 = double layer <x-y, n_y>/(4 pi r^3)
     * (assembly.py:196-201) */
    int64_t kernel;
    /* linear basis (basis = 1): per vertex v the star entries
     * vstar_ent[vstar_ptr[v] .. vstar_ptr[v+1]) = (triangle << 2 | corner)
     * ordered by (corner, triangle) - the order in which the reference's
     * np.add.at scatters a vertex's moments (assembly.py:406-415) - and the
     * barycentric values bq [dev] (mq x 3) of the regular rule's points */
    const int64_t* vstar_ptr;
    const int64_t* vstar_ent;
    const double* bq;
    /* 0 = piecewise constant, 1 = piecewise linear, 2 = collocation rows
     * (point evaluations at the vertices, Green factors only) */
    int64_t basis;
    const double* verts;   /* [dev] nv x 3 vertex coordinates (collocation) */
    /* curved (quadratic) charts, all NULL for plane charts (geometry.py:
     * 266-293): nodes6 / nrm6 [dev] nt x 6 x 3 chart nodes and node normals,
     * gq [dev] nt x mq Gramians |n| at the regular points, nq [dev] nt x mq
     * x 3 the interpolated normals there (double layer) */
    const double* nodes6;
    const double* nrm6;
    const double* gq;
    const double* nq;
} gc_geom;

/* Singular pair rules (quadrature.sauter_rule, quadrature.py:211-284) in
 * the xi-reduced form of quadrature.reduced_sauter_rule: SoA tables [dev]
 * of (NC+1)*P doubles, NC coefficient columns then the weights, with
 * D = sum_k coef_k G_k; NC = 4 (vertex: E1,E2,-F1,-F2), 3 (edge: E1,E2,-F2),
 * 2 (identical: E1,E2).  npts[c] = P. */
typedef struct gc_rules {
    const double* table[4]; /* index by case code; [0] unused */
    int64_t npts[4];
} gc_rules;

/* Quadrature points of the regular rule on every chart, in the reference's
 * exact operation order: xq[t,m,c] = sum_a n6[m,a] node[t,a,c] summed
 * sequentially without FMA, nodes = corners + straight midpoints
 * (assembly._interp6 / _surface_quadrature, assembly.py:138-143, 371-381).
 *   n6 [dev] (mq,6) shape functions at the triangle_gauss(q_reg) points. */
/* Plane chart data and cluster support of every triangle, bit-identical to
 * the host's numpy arrays (geometry.py:266-293 chart_pack, :324-338
 * control_points, clustering.py:107-128 support boxes, centroids): verts
 * [dev] (nv,3), tris [dev] (nt,3), gu / gv [host] (6) = the shape-function
 * gradients at node 0 -> corners [dev] (nt,3,3), gram [dev] (nt), normal
 * [dev] (nt,3) (|normal| = gram), support [dev] (nt,9) = control-point box
 * lower | upper | centroid. */
int gc_chart_pack(const double* verts, const int64_t* tris, int64_t nt, const double* gu, const double* gv,
                  double* corners, double* gram, double* normal, double* support, void* stream);
int gc_surface_points(const double* corners, int64_t nt, const double* n6,
                      int64_t mq, double* xq, void* stream);

/* Batched pair quadrature for the evaluator seam: replaces the evaluator
 * galerkin_pair_evaluator(...).evaluate(case, rows, cols, px, py)
 * (assembly.py:159-216; contract batchexec.py:70-76, 161-163).
 *   rows, cols, px, py [dev] (B,) int64; out [dev] (B,) double.
 * Constant basis, plane charts, single layer. */
int gc_pair_eval(const gc_geom* g, const gc_rules* r, int kase, int64_t B,
                 const int64_t* rows, const int64_t* cols, const int64_t* px,
                 const int64_t* py, double* out, void* stream);

/* Singular-task queues filled by gc_assemble_blocks: per case c in 1..3 a
 * [dev] array of cap[c] packed tasks (t, s, px | py << 8, out_index). */
typedef struct gc_queue {
    int64_t* tasks[4];
    int64_t cap[4];
    int32_t* count; /* [dev] 4 counters */
} gc_queue;

/* Whole-block Galerkin assembly (replaces the executor path of
 * gca.build_h2, gca.py:282-312, for near-field and coupling blocks and
 * assembly.assemble_galerkin_block, assembly.py:330-337).
 * desc [dev] (nb,5) int64: row_off, nr, col_off, nc, out_off.  Entry (a,b)
 * pairs triangle row_idx[row_off+a] with col_idx[col_off+b] and is stored
 * column-major at out[out_off + b*nr + a].  Disjoint pairs are integrated
 * here; singular pairs are appended to the queue and integrated by
 * gc_singular_flush.  max_rows / max_cols bound nr / nc over the batch
 * (shared-memory staging).  flags [dev] int: bit 1 set on queue overflow. */
int gc_assemble_blocks(const gc_geom* g, int64_t nb, const int64_t* desc,
                       int64_t max_rows, int64_t max_cols, const int64_t* row_idx,
                       const int64_t* col_idx, double* out, gc_queue* q,
                       int32_t* flags, void* stream);

/* Integrate all queued singular tasks into out and reset the counters.
 * Synchronises `stream` once to read the counters; counts [host] (4,)
 * receives the number of tasks per case (index 1..3; may be NULL). */
int gc_singular_flush(const gc_geom* g, const gc_rules* r, gc_queue* q,
                      double* out, int64_t* counts, void* stream);

/* gc_singular_flush without the host synchronisation: the singular kernels
 * read their task counts from the queue's device counters (clamped to the
 * capacity; an overflow sets the gc_assemble_blocks flag), then the
 * counters are copied to counts_dev [dev] (4 x int32, may be NULL) and
 * reset, all in stream order.  Plane charts only. */
int gc_singular_flush_async(const gc_geom* g, const gc_rules* r, gc_queue* q,
                            double* out, int32_t* counts_dev, void* stream);

/* Block tree (replaces clustering.build_block_tree / admissible,
 * clustering.py:215-237), host memory only: row and column cluster trees
 * as flat preorder arrays (diam (n), lower / upper (n,3), left / right with
 * -1 at leaves), the two roots, eta, the rounding sequence of the 1-D BLAS
 * norm used to re-decide near ties (0 / 1, see gc_host_norm3) and the key
 * width in base-4 digits.  Builds the nodes in build order (level by level;
 * children grouped by child slot, then by parent): row, col, state (0
 * admissible, 1 inadmissible leaf, 2 subdivided), level, key, parent; they
 * are held by *handle, *count = number of nodes.  gc_block_tree_fetch
 * copies them into caller arrays (any may be NULL) and frees the handle. */
int gc_block_tree(const double* r_diam, const double* r_lower, const double* r_upper,
                  const int64_t* r_left, const int64_t* r_right, const double* c_diam,
                  const double* c_lower, const double* c_upper, const int64_t* c_left,
                  const int64_t* c_right, int64_t root_r, int64_t root_c, double eta,
                  int32_t norm_mode, int32_t digits, void** handle, int64_t* count);
int gc_block_tree_fetch(void* handle, int64_t* row, int64_t* col, int8_t* state, int64_t* level,
                        int64_t* key, int64_t* parent);

/* The same block tree built on the device one level per gc_bt_level call
 * (below): the frontier pairs fr, fc, fkey, fpar [dev] are decided
 * (gc_block_tree's rounding) and recorded at out_*[base ..] [dev]; their
 * children go to nr, nc, nk, np [dev] in gc_block_tree's order.  Tree
 * arrays [dev] as gc_block_tree; temp [dev] of gc_bt_level_bytes(cap_f). */
int gc_bt_level_bytes(int64_t cap_f, int64_t* bytes);
/* The leaves of a device block tree (n nodes, state / key [dev]) in
 * depth-first order: leaf_ids, leaf_key [dev] (capacity n), *count [dev].
 * Scratch [dev]: ids, ids_sorted, key_sorted (n int64), flag, flag_sorted
 * (n bytes), temp of gc_bt_leaves_bytes(n) bytes. */
int gc_bt_leaves_bytes(int64_t n, int64_t* bytes);
int gc_bt_leaves(int64_t n, const int8_t* state, const int64_t* key, int64_t* leaf_ids, int64_t* leaf_key,
                 int64_t* count, int64_t* ids, int64_t* ids_sorted, int64_t* key_sorted, char* flag,
                 char* flag_sorted, void* temp, int64_t temp_bytes, void* stream);
/* One level of the same build on the device, no host read: meta [dev] =
 * (frontier size, node offset) of this level, the next level's written to
 * meta[2..3]; frontier / next frontier capacity cap_f, node capacity cap_n;
 * flags / pos [dev] 4 cap_f int32; err [dev] int32 bits: 1 frontier, 2 node
 * capacity, 4 key digits exhausted (the tree then ends at this level). */
int gc_bt_level(int64_t* meta, int64_t cap_f, int64_t cap_n, const int64_t* fr, const int64_t* fc,
                const int64_t* fkey, const int64_t* fpar, int64_t lev, int32_t digits, const double* r_diam,
                const double* r_lower, const double* r_upper, const int64_t* r_left, const int64_t* r_right,
                const double* c_diam, const double* c_lower, const double* c_upper, const int64_t* c_left,
                const int64_t* c_right, double eta, int32_t norm_mode, int64_t* o_row, int64_t* o_col,
                int8_t* o_state, int64_t* o_level, int64_t* o_key, int64_t* o_parent, int64_t* nr, int64_t* nc,
                int64_t* nk, int64_t* np, int32_t* flags, int32_t* pos, int32_t* err, void* temp,
                int64_t temp_bytes, void* stream);

/* Level bookkeeping of the nested bases (replaces the host loop body of
 * greencross gca.py:162-220 around the factor / ACA launches).  Per basis
 * side, tree arrays left/right/start/stop, rank/piv_off/rows/v_off per tree
 * node and the global pivots gpiv with a device cursor stay on the device.
 * gc_bases_R: factor rows R (leaf size or sum of the children's ranks),
 * min(R, W) and R*min(R, W) of the n nodes at level positions pos0...
 * gc_bases_scan: exclusive scans of those over the level's nn nodes and
 * out = [max R, rows, limits, vcap, v_off at the n_bound positions bounds].
 * gc_bases_rows: row lists (leaf dofs from perm, or the children's
 * pivots) and the gc_green_factor (5 per node) / gc_aca (4) descriptors.
 * gc_bases_post: after gc_aca, ranks, compact global pivots, piv_off and
 * v_off (v_base + level offset) of one side; rk_off (n) and temp scratch. */
int gc_bases_scan_bytes(int64_t nn, int64_t* bytes);
int gc_bases_R(int64_t n, const int64_t* nodes, const int64_t* left, const int64_t* right, const int64_t* start,
               const int64_t* stop, const int64_t* rank, int64_t pos0, int64_t W, int64_t* R, int64_t* lim,
               int64_t* vcap, int64_t* rows_node, void* stream);
int gc_bases_scan(int64_t nn, const int64_t* R, const int64_t* lim, const int64_t* vcap, int64_t* rows_off,
                  int64_t* piv_off_l, int64_t* v_off, const int64_t* bounds, int64_t n_bound, int64_t* out,
                  void* temp, int64_t temp_bytes, void* stream);
int gc_bases_rows(int64_t n, const int64_t* nodes, const int64_t* left, const int64_t* right, const int64_t* start,
                  const int64_t* rank, const int64_t* piv_off, const int64_t* gpiv, const int64_t* perm, int64_t pos0,
                  int64_t box0, int64_t side, int64_t W, const int64_t* R, const int64_t* rows_off,
                  const int64_t* piv_off_l, const int64_t* v_off, int64_t* rows, int64_t* fdesc, int64_t* adesc,
                  void* stream);
int gc_bases_post(int64_t n, const int64_t* nodes, int64_t pos0, const int64_t* rank_l, const int64_t* piv_l,
                  const int64_t* piv_off_l, const int64_t* rows, const int64_t* rows_off, const int64_t* v_off,
                  int64_t v_base, int64_t* cursor, int64_t* rank, int64_t* piv_off, int64_t* gpiv,
                  int64_t* v_off_node, int64_t* rk_off, void* temp, int64_t temp_bytes, void* stream);

/* Block tables of build_h2 (gca.py:282-312: the admissible leaves become
 * coupling blocks, pivot rows x pivot columns, the inadmissible ones
 * near-field blocks, full clusters).  From nl block-tree leaves leaf_ids
 * [dev] in depth-first order with node_row / node_col [dev] (int64) and
 * node_state [dev] (int8, 0 admissible / 1 inadmissible), the blocks of
 * one kind (near = 0 coupling, 1 near field), optionally only block rows
 * whose cluster lies in tree positions [lo, hi) (lo < 0: all).  Sizes are
 * the ranks r_rank / c_rank [dev] (coupling) or the cluster sizes from
 * r_start / r_stop / c_start / c_stop [dev]; a coupling block whose row
 * cluster has r_ok = 0 or column cluster c_ok = 0 [dev] (int8: basis content
 * / pivots present) is counted in totals[7].  Storage offsets group the
 * blocks by key = row cluster (sharded: 2 row + column outside [lo, hi)),
 * stable in DFS order, keys below 2^key_bits - 1.
 * table [dev] (6 x count, column-major with stride count): row, col, nr,
 * nc, off, order (block indices by ascending offset); desc [dev] (count x 5)
 * of the non-empty blocks for gc_assemble_blocks: (row_off, nr, col_off,
 * nc, off) with row/col offsets into the pivot lists r_poff / c_poff
 * (coupling) or the cluster starts (near); totals [dev] (8 int64, zeroed
 * by the caller): count, non-empty, max nr, max nc, entries, two counters,
 * blocks without basis content.  Scratch [dev]: 12 nl
 * int64, 2 nl bytes, temp of gc_h2_blocks_bytes(nl) bytes.  No host sync. */
int gc_h2_blocks_bytes(int64_t nl, int64_t* bytes);
int gc_h2_blocks(int64_t nl, const int64_t* leaf_ids, const int64_t* node_row, const int64_t* node_col,
                 const int8_t* node_state, const int64_t* r_start, const int64_t* r_stop, const int64_t* c_start,
                 const int64_t* c_stop, const int64_t* r_rank, const int64_t* r_poff, const int64_t* c_rank,
                 const int64_t* c_poff, const int8_t* r_ok, const int8_t* c_ok, int64_t lo, int64_t hi,
                 int32_t near, int32_t key_bits, int64_t* table, int64_t* desc, int64_t* totals, int64_t* scratch,
                 char* flags, void* temp, int64_t temp_bytes, void* stream);

/* Batched transpose: for node i with desc (off, rows, cols) [dev] (nn,3):
 * out[off + c*rows + r] = in[off + r*cols + c]. */
int gc_batched_transpose(int64_t nn, const int64_t* desc, const double* in,
                         double* out, void* stream);

/* Box-boundary Green rules of a batch of cluster boxes: replaces
 * quadrature.green_box_rule (quadrature.py:95-126) evaluated per node.
 *   g01, w01 [dev] (m,) Gauss-Legendre on [0,1];
 *   box [dev] (nn,8) double: lower[3], upper[3], delta, d_tau (host values);
 *   outputs [dev]: z (nn,K,3) points, sq (nn,K) sqrt(weights), nz (nn,K,3)
 *   outward normals; K = 6 m^2. */
int gc_green_box_rules(int m, const double* g01, const double* w01, int64_t nn,
                       const double* box, double* z, double* sq, double* nz,
                       void* stream);

/* Green quadrature factors for a batch of cluster-basis nodes: replaces
 * assembly.green_row_factor / green_col_factor (assembly.py:420-455).
 *   side 0: A = [sqrt(w) g, -d sqrt(w) h];  side 1: B = [sqrt(w) h, sqrt(w)/d g]
 *   desc [dev] (nn,5) int64: rows_off, R, out_off, rule index, side;
 *   side -1 takes the side per node from desc (one launch for both bases);
 *   dtau [dev] (nn,) box diameters (host values); z/sq/nz: rules as above;
 *   rows [dev] dof (triangle) ids; out [dev] row-major (R, 2K) per node.
 * flags bit 0 is set when an expansion point touches the surface
 * (r <= 1e-12, assembly._touch_guard, assembly.py:365-368). */
int gc_green_factor(const gc_geom* g, int side, int64_t K, int64_t nn,
                    const int64_t* desc, const double* dtau, const double* z,
                    const double* sq, const double* nz, const int64_t* rows,
                    double* out, int32_t* flags, void* stream);

/* Batched full-pivot cross approximation (gca.aca_interpolation,
 * gca.py:41-79) of nn thin matrices of width W.
 *   desc [dev] (nn,4) int64: fac_off, R, piv_off, v_off.  The factor at
 *   fac[fac_off] (R x W row-major) is overwritten.  Outputs: rank[n],
 *   piv[piv_off + k] local pivot rows (k < rank), V at v[v_off] (R x rank
 *   row-major, V[piv] = I exactly); u is scratch of the same layout as v.
 *   max_rank <= 0 means W.  max_rows bounds R over the batch. */
int gc_aca(int64_t nn, const int64_t* desc, int64_t W, double eps,
           int64_t max_rank, double* fac, int64_t* piv, int64_t* rank,
           double* v, double* u, int64_t max_rows, void* stream);

/* ---------------------------------------------------------------------
 * H2 matvec building blocks (h2.mvm, h2.py:19-80)
 * ------------------------------------------------------------------- */
/* xt[i] = x[perm[i]] (h2.py:68) */
int gc_gather(const double* x, const int64_t* perm, int64_t n, double* xt,
              void* stream);
/* y[perm[i]] = yt[i] (h2.py:78-79) */
int gc_scatter(const double* yt, const int64_t* perm, int64_t n, double* y,
               void* stream);
/* The same indexed from the external side, iperm = inverse permutation:
 * xt[iperm[j]] = x[j] and y[j] = yt[iperm[j]] + yt2[iperm[j]] - contiguous
 * in x / y, so those may be mapped pinned host memory. */
int gc_gather_inv(const double* x, const int64_t* iperm, int64_t n, double* xt, void* stream);
int gc_scatter2_inv(const double* yt, const double* yt2, const int64_t* iperm, int64_t n, double* y,
                    void* stream);
/* y[perm[i]] = yt[i] + yt2[i] (the panel plan's two output parts) */
int gc_scatter2(const double* yt, const double* yt2, const int64_t* perm, int64_t n, double* y,
                void* stream);
/* out[off[s] + j] = start[s] + j for j < len[s]: index ranges expanded to a
 * panel phase's input index list (int32) */
int gc_expand_ranges(int64_t m, const int64_t* start, const int64_t* len, const int64_t* off,
                     int32_t* out, void* stream);
/* Re-point argument `arg` of the gather (kernel 0, gc_gather; 2,
 * gc_gather_inv) or scatter (kernel 1, gc_scatter2; 3, gc_scatter2_inv) kernel nodes of an instantiated CUDA graph whose
 * captured value is old_ptr to new_ptr in the executable graph
 * (cudaGraphExecKernelNodeSetParams; the graph itself keeps old_ptr): a captured
 * product reads / writes caller buffers without copies.  graph / exec =
 * cudaGraph_t / cudaGraphExec_t; *count = nodes updated. */
int gc_graph_retarget(void* graph, void* exec, int32_t kernel, int32_t arg, const void* old_ptr,
                      const void* new_ptr, int32_t* count);

/* Panel product, the mvm hot path (one phase of h2.py:63-80).  A phase
 * is a list of work items; item i (items[8i..8i+7] = a_off, xi_off,
 * out_off, T, nrows, mode, red_slot, 0) computes
 *     s[t] = sum_{r < nrows} A[a_off + r*T + t] * in[xidx[xi_off + r]]
 * over a contiguous row-major chunk of a panel (A = A1 if mode&1, in = in1
 * if mode&2; in = in0 + in1 if mode&32) and writes s to out[out_off + t]
 * (mode&4; added to it if mode&8) or, for a panel split over several
 * items, to scratch[out_off+t].
 * red (nred,5) = out_off, T, scratch_off, nitems, accumulate describes each
 * split panel; the last item of a panel to finish (arrivals[red_slot], an
 * int32 counter that must start at 0 and is re-armed by the kernel) sums
 * the scratch rows into out in item order.  One writer per output, fixed
 * order: deterministic.  chain & 1 launches with programmatic stream
 * serialization (PDL): the kernel prefetches its matrix chunk while the
 * previous kernel on the stream drains and waits for it before reading in
 * (for the latency-bound transform levels); the next launch is released at
 * each CTA's start.  chain & 16 runs two whole small panels per CTA (direct
 * items, T <= 128, <= 512 rows).  chain & 32 streams each item's matrix
 * through a 2-stage shared-memory ring of 1-D TMA bulk copies issued before
 * the input gather (bulk phases, T <= 256; the matrix buffer must be
 * readable 16 bytes past its end); same results bit for bit.  priority != 0 sets the
 * launch's scheduling priority (CUDA stream-priority scale, lower = more
 * urgent; 0 = the stream's own).  trace (optional, NULL = off)
 * = [dev] 2 x uint64 receiving min(start) / max(end) %globaltimer (ns) of
 * the launch's CTAs, for timelines inside CUDA graphs. */
int gc_panelmv(int64_t nitems, const int64_t* items, const int32_t* xidx,
               const double* A0, const double* A1, const double* in0,
               const double* in1, double* out, double* scratch, int64_t nred,
               const int64_t* red, int32_t* arrivals, int32_t chain, int32_t priority,
               uint64_t* trace, void* stream);

/* Native product executor (h2.py:63-80 as one call).  nodes [host] (n,18)
 * int64 rows: kind (0 panel phase, 1 memset, 2 gc_gather_inv,
 * 3 gc_scatter2_inv, 4 NCCL all-gather), stream index, launch priority,
 * chain flags (as gc_panelmv), ndeps, dep_off, then 12 arguments: panel =
 * items, nitems, xidx, A0, A1, in0, in1, out, scratch, nred, red,
 * arrivals; memset = ptr, bytes; gather = x, iperm, n, xt; scatter = yt,
 * yt2, iperm, n, y; all-gather = send, recv, count, communicator
 * (gc_nccl_comm_init) - the block-row sharded product is one
 * such plan per rank: the own slice of x gathered in, the x and x-hat
 * all-gathers, the product, the own rows of y scattered out.  deps
 * [host] = dependency node indices (each earlier than its node).
 * stream_prio [host] (nstreams) = stream creation priorities.  Captures the
 * DAG on the plan's own streams/events into one CUDA graph and
 * instantiates it.  gc_plan_run re-points the gather / scatter nodes at x /
 * y (device or mapped pinned host, external order; NULL keeps the binding)
 * and launches the graph on `stream`. */
int gc_plan_create(int64_t n, const int64_t* nodes, int64_t ndeps, const int64_t* deps, int64_t nstreams,
                   const int32_t* stream_prio, void** plan);
int gc_plan_run(void* plan, const double* x, double* y, void* stream);
/* h2.mvm in one call: copies n_in doubles of host x into the pinned
 * staging buffer x_pinned, runs the plan reading x_pinned and writing the
 * pinned y_pinned over the host link, and synchronises `stream`. */
int gc_plan_run_host(void* plan, const double* x_host, double* x_pinned, int64_t n_in, double* y_pinned,
                     void* stream);
int gc_plan_destroy(void* plan);

/* Tiered transforms (plan time; h2.py PanelPlan tiers): the composed
 * transfers of a tier of tree heights, one height per call.  desc [dev]
 * (n,6) = s_off, m, kc, e_off, ku, out_off, cut into tiles [dev] (ntiles,2)
 * = descriptor index, first output entry (every gc_tier_tile() entries of
 * each descriptor's m x ku block):
 *     M[out_off..] (m x ku) = M[s_off..] (m x kc) @ V[e_off..] (kc x ku)
 * or, s_off < 0, a copy of the m x ku block V[e_off..] (row-major, each
 * entry summed over kc in order).  gc_block_transpose: desc [dev] (n,5) =
 * src_off, ld, rows, cols, dst_off: dst[dst_off + c*rows + r] =
 * src[src_off + r*ld + c] (the backward transform's regrouped blocks).
 * Follows the nested-basis recursion of gca.py:162-220 multiplied out. */
int gc_tier_compose(int64_t ntiles, const int64_t* tiles, const int64_t* desc, const double* V,
                    double* M, void* stream);
int64_t gc_tier_tile(void);
int gc_block_transpose(int64_t n, const int64_t* desc, const double* src, double* dst,
                       void* stream);

/* Piecewise-linear basis (assembly.py:54-135, 175-214, 279-304;
 * batchexec.py:178-209).  gc_lin_pairs: tasks [dev] (n,2) triangle pairs
 * (t, s); for each, 9 pair integrals of k(x,y) phi_a(x) phi_c(y) in the
 * canonical permuted local order -> U[9i..9i+8], pp[i] = px | py << 8;
 * disjoint pairs integrate the regular rule (rule_w [host] q^2 weights,
 * rule_b [host] q^2 x 3 barycentric values), singular pairs are queued.
 * gc_lin_singular: integrates the queued pairs with the reference's full
 * Sauter-Schwab rules (r->table[c] = SoA x1, x2, y1, y2, w of npts[c]
 * points).  gc_lin_gather: desc (nb,7) = row_ptr_off, nr, col_ptr_off, nc,
 * out_off, task_base, n_col_tris; rptr/cptr CSR per DOF into rlist/clist
 * of packed (table_row << 2 | corner); out column-major per block, each
 * entry the fixed-order sum of its pairs' contributions. */
int gc_lin_pairs(const gc_geom* g, const double* rule_w, const double* rule_b, int64_t n,
                 const int64_t* tasks, double* U, int32_t* pp, gc_queue* q, int32_t* flags,
                 void* stream);
int gc_lin_singular(const gc_geom* g, const gc_rules* r, gc_queue* q, double* U,
                    int64_t* counts_out, void* stream);
int gc_lin_gather(int64_t nb, const int64_t* desc, const int64_t* rptr, const int64_t* rlist,
                  const int64_t* cptr, const int64_t* clist, const double* U, const int32_t* pp,
                  double* out, void* stream);
/* gc_lin_pairs over blocks without materialising the pair list: pair i
 * belongs to the block b with the last blk[4b] (task_base) <= i (ascending),
 * blk (nblk,4) = task_base, n_col_tris, row table offset, column table
 * offset; local = i - task_base -> (tri_r[row_off + local / n_col_tris],
 * tri_c[col_off + local % n_col_tris]). */
int gc_lin_pairs_blocks(const gc_geom* g, const double* rule_w, const double* rule_b, int64_t n,
                        int64_t nblk, const int64_t* blk, const int64_t* tri_r, const int64_t* tri_c,
                        double* U, int32_t* pp, gc_queue* q, int32_t* flags, void* stream);

/* Singular pairs of curved charts: the queued tasks (from
 * gc_assemble_blocks / gc_lin_pairs) integrated with the full Sauter-Schwab
 * rules r->table[c] = SoA (x1, x2, y1, y2, w), charts and Gramians
 * evaluated per point; width 1 (constant basis) or 9 (linear basis). */
int gc_curved_singular(const gc_geom* g, const gc_rules* r, gc_queue* q, int64_t width,
                       double* out, int64_t* counts_out, void* stream);
/* The same for an explicit task list (t, s, px | py << 8, out index) [dev]
 * and one rule [dev] (SoA x1, x2, y1, y2, w, P points): the evaluator seam
 * on curved charts. */
int gc_curved_pairs(const gc_geom* g, const double* rule, int64_t P, const int64_t* tasks, int64_t n,
                    int64_t width, double* out, void* stream);

/* Collocation (assembly.py:219-276, 340-362): tasks (n,2) = (vertex v,
 * triangle s); each the 3 single integrals of k(x_v, y) phi_c(y) over s
 * (regular rule: the gc_geom chart points; v a corner of s: the collapsed
 * Gauss rule sing_w / sing_p (ms points) with v rotated to corner 0) in
 * the rotated column order -> U[9i .. 9i+2], pp[i] = rotation << 8, the
 * layout gc_lin_gather reads. */
int gc_col_pairs(const gc_geom* g, const double* verts, const double* reg_w, const double* reg_b,
                 int64_t ms, const double* sing_w, const double* sing_p, int64_t n,
                 const int64_t* tasks, double* U, int32_t* pp, void* stream);
/* gc_col_pairs over blocks (pair derivation as gc_lin_pairs_blocks, rows
 * are points pts_r); nsing [dev] counts the singular (corner) pairs. */
int gc_col_pairs_blocks(const gc_geom* g, const double* verts, const double* reg_w, const double* reg_b,
                        int64_t ms, const double* sing_w, const double* sing_p, int64_t n, int64_t nblk,
                        const int64_t* blk, const int64_t* pts_r, const int64_t* tri_c, double* U,
                        int32_t* pp, int32_t* nsing, void* stream);

/* Cluster-tree construction per depth (clustering.py:131-162): segmented
 * support boxes box[6s..6s+5] = (min lo, max hi) over rows [start, stop)
 * of pack [dev] (n x 9 = lo | hi | point); and one split step - the split
 * coordinate of each dof of each splitting segment (start, len, head,
 * axis [dev] each nseg int64; offsets [dev] nseg+1 int32 = head and end),
 * a stable segmented sort (CUB), and pack_new[pos] = pack_old[src],
 * perm_new[pos] = perm_old[src] (the *_new buffers start as copies);
 * scratch keys (2 nitems doubles), vals (2 nitems int32) and temp
 * (gc_tree_sort_bytes) are caller-owned device memory. */
int gc_tree_boxes(int64_t nseg, const int64_t* start, const int64_t* stop, const double* pack,
                  double* box, void* stream);
int gc_tree_sort_bytes(int64_t nitems, int64_t nseg, int64_t* bytes);
/* Split axes: axis[i] = argmax of the extents of box row rows[i] (first
 * maximum; clustering.py:154 np.argmax(box.upper - box.lower)). */
int gc_tree_axis(int64_t k, const int64_t* rows, const double* box, int64_t* axis, void* stream);
/* gc_tree_split for a depth whose segments are all short: one stable
 * segmented sort over the offsets (required here) instead of two radix
 * sorts; identical result.  gc_tree_sort_bytes(nitems, nseg) covers both. */
int gc_tree_split_small(int64_t nseg, const int64_t* seg_start, const int64_t* seg_len, const int64_t* seg_head,
                        const int64_t* seg_axis, const int32_t* offsets, int64_t nitems, const double* pack_old,
                        double* pack_new, const int64_t* perm_old, int64_t* perm_new, double* keys, int32_t* vals,
                        void* temp, int64_t temp_bytes, void* stream);
int gc_tree_split(int64_t nseg, const int64_t* seg_start, const int64_t* seg_len, const int64_t* seg_head,
                  const int64_t* seg_axis, const int32_t* offsets, int64_t nitems, const double* pack_old,
                  double* pack_new, const int64_t* perm_old, int64_t* perm_new, double* keys, int32_t* vals,
                  void* temp, int64_t temp_bytes, void* stream);

/* Device-side Krylov support (consumers of the matvec, h2.py:190-253;
 * SURVEY 8f rank 3).  Deterministic dot product: fixed grid of
 * gc_krylov_partials() blocks, `partial` [dev] holds that many doubles.
 * gc_dot: out[0] = a.b.  CG state s [dev, 8 doubles]: s[0] = r.r, s[1] =
 * p.q, s[2] = new r.r, s[3] = beta, s[4] = alpha, s[5] = stop flag.
 * gc_cg_pq: s[1] = p.q.  gc_cg_update: alpha = s[0]/s[1]; x += alpha p;
 * r -= alpha q; s[2] = r.r; beta = s[2]/s[0]; s[0] = s[2]; p = r + beta p
 * (p.q <= 0 sets s[5] = 1 and leaves x, r unchanged, as h2.py:206-208). */
int gc_dot(int64_t n, const double* a, const double* b, double* partial, double* out, void* stream);
int gc_cg_pq(int64_t n, const double* p, const double* q, double* partial, double* s, void* stream);
int gc_cg_update(int64_t n, double* x, double* r, double* p, const double* q, double* partial,
                 double* s, void* stream);
int64_t gc_krylov_partials(void);
/* CGNR (h2.py:222-253), state s [dev, 8 doubles]: [0] s.s, [1] q.q, [2] r.r,
 * [3] beta, [4] new s.s, [5] stop flag.  gc_cgnr_step: q.q; stop (s[5] = 1,
 * x and r unchanged) if it is 0, else alpha = s[0] / q.q, x += alpha p,
 * r -= alpha q; then s[2] = r.r.  gc_cgnr_dir: s[4] = sv.sv, beta =
 * s[4] / s[0], p = sv + beta p, s[0] = s[4]. */
int gc_cgnr_step(int64_t n, double* x, double* r, const double* p, const double* q, double* partial,
                 double* s, void* stream);
int gc_cgnr_dir(int64_t n, const double* sv, double* p, double* partial, double* s, void* stream);
/* Power iteration (h2.py:144-184): z /= sqrt(s[0]); b -= a. */
int gc_scale_inv_norm(int64_t n, double* z, const double* s, void* stream);
int gc_axpy_neg(int64_t n, const double* a, double* b, void* stream);

/* NCCL for the sharded product (SURVEY 8b gc_nccl_init), resolved at run
 * time (libnccl.so.2; inside a torch process torch's own copy).
 * gc_nccl_unique_id: id [host] 128 bytes (rank 0 creates it, every rank
 * receives it out of band).  gc_nccl_comm_init: with the rank's device
 * current; *comm = the communicator.  gc_nccl_all_gather: recv [dev]
 * (nranks * count doubles) = concatenation of every rank's send [dev]
 * (count doubles); in place when send = recv + rank * count. */
int gc_nccl_unique_id(void* id);
int gc_nccl_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm);
int gc_nccl_comm_destroy(void* comm);
int gc_nccl_all_gather(const double* send, double* recv, int64_t count, void* comm, void* stream);

/* The device's scheduling-priority range (cudaDeviceGetStreamPriorityRange):
 * least (default, e.g. 0) and greatest (most urgent, e.g. -5). */
int gc_priority_range(int32_t* least, int32_t* greatest);

/* Host helper (no device): norms of n 3-vectors v [host] (n,3) into out
 * [host] (n,) with mode 0 = sqrt(fma(z,z,fma(y,y,x*x))) (the rounding of
 * numpy's 1-D norm through OpenBLAS ddot, used for box diameters,
 * clustering.py:34-43) or mode 1 = sqrt((x*x+y*y)+z*z). */
int gc_host_norm3(const double* v, int64_t n, double* out, int mode);

/* FP64 DFMA throughput probe used as the roofline denominator (no FP64
 * figure exists in MEASURED_PEAKS.json): blocks x threads x iters x 8 DFMA. */
int gc_dfma_probe(int64_t blocks, int64_t threads, int64_t iters, double* out,
                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GCB200_H */

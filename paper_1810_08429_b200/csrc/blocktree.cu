// Block tree (clustering.py:215-237 build_block_tree / admissible) built on
// the host in one native pass, level by level in the same node order as the
// array-at-a-time Python builder (clustering.build_block_tree): frontier
// pairs in order, admissibility decided bit for bit like the reference, then
// the children of every subdivided pair appended grouped by child slot
// (row child a, column child b; a-major) and, inside a group, by parent.
// Host code only; no device memory involved.
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"

namespace {

// numpy's elementwise sqrt((g0*g0 + g1*g1) + g2*g2): every product and sum
// rounds separately (volatile: no contraction whatever the host flags)
double norm3_plain(double a, double b, double c) {
    volatile double aa = a * a, bb = b * b, cc = c * c;
    volatile double s = (double)aa + (double)bb;
    return std::sqrt((double)s + (double)cc);
}

// the 1-D numpy norm (np.linalg.norm of a 3-vector) in the rounding
// sequence gc_host_norm3 reproduces (mode found by clustering.blas_norms)
double norm3_blas(double x, double y, double z, int mode) {
    volatile double xx = x * x;
    if (mode == 0) return std::sqrt(std::fma(z, z, std::fma(y, y, (double)xx)));
    volatile double yy = y * y, zz = z * z;
    volatile double t = (double)xx + (double)yy;
    return std::sqrt((double)t + (double)zz);
}

struct Tree {
    const double* diam;
    const double* lower;   // (n,3)
    const double* upper;
    const int64_t* left;
    const int64_t* right;
};

// clustering._admissible_many for one pair
bool admissible(const Tree& R, const Tree& C, int64_t r, int64_t c, double eta, int mode) {
    const double d = R.diam[r] > C.diam[c] ? R.diam[r] : C.diam[c];
    double g[3];
    for (int k = 0; k < 3; ++k) {
        const double a = R.lower[3 * r + k] - C.upper[3 * c + k];
        const double b = C.lower[3 * c + k] - R.upper[3 * r + k];
        const double m = a >= b ? a : b;                     // np.maximum (only squares are used)
        g[k] = m >= 0.0 ? m : 0.0;
    }
    const double two_eta = 2.0 * eta;
    const double rhs = two_eta * norm3_plain(g[0], g[1], g[2]);
    const double big = d > rhs ? d : rhs;
    if (std::fabs(d - rhs) <= 1e-12 * big) return d <= two_eta * norm3_blas(g[0], g[1], g[2], mode);
    return d <= rhs;
}

struct BlockTreeOut {
    std::vector<int64_t> row, col, level, key, parent;
    std::vector<int8_t> state;
};

}  // namespace

extern "C" {

// Block tree of a row and a column cluster tree (flat preorder arrays,
// clustering.FlatClusterTree: diam (n), lower / upper (n,3), left / right
// (-1 at leaves)).  Builds every node in build order: row, col, state (0
// admissible, 1 inadmissible leaf, 2 subdivided), level, key (base-4 path
// digits aligned to `digits`), parent (-1 for the root), held by *handle;
// *count = number of nodes.  gc_block_tree_fetch copies them out and frees
// the handle.
int gc_block_tree(const double* r_diam, const double* r_lower, const double* r_upper, const int64_t* r_left,
                  const int64_t* r_right, const double* c_diam, const double* c_lower, const double* c_upper,
                  const int64_t* c_left, const int64_t* c_right, int64_t root_r, int64_t root_c, double eta,
                  int32_t norm_mode, int32_t digits, void** handle, int64_t* count) {
    using namespace gcb;
    if (!r_diam || !r_lower || !r_upper || !r_left || !r_right || !c_diam || !c_lower || !c_upper || !c_left ||
        !c_right || !count || !handle || eta <= 0.0 || (norm_mode != 0 && norm_mode != 1) || digits < 1 ||
        digits > 31) {
        set_error(GC_ERR_CONFIG, "gc_block_tree: bad arguments");
        return GC_ERR_CONFIG;
    }
    *handle = nullptr;
    const Tree R{r_diam, r_lower, r_upper, r_left, r_right};
    const Tree C{c_diam, c_lower, c_upper, c_left, c_right};
    BlockTreeOut* o = new BlockTreeOut();
    const size_t guess = 64 * (size_t)(root_r + 1) + 4096;
    o->row.reserve(guess); o->col.reserve(guess); o->state.reserve(guess);
    o->level.reserve(guess); o->key.reserve(guess); o->parent.reserve(guess);
    std::vector<int64_t> fr{root_r}, fc{root_c}, fkey{0}, fpar{-1};
    std::vector<int64_t> nr, nc, nk, np_;
    std::vector<int64_t> sub;
    int64_t base = 0, lev = 0;
    while (!fr.empty()) {
        if (lev >= digits) {
            delete o;
            set_error(GC_ERR_CONFIG, "block tree deeper than %d levels", digits);
            return GC_ERR_CONFIG;
        }
        const int64_t m = (int64_t)fr.size();
        sub.clear();
        for (int64_t i = 0; i < m; ++i) {
            const int64_t r = fr[i], c = fc[i];
            const bool adm = admissible(R, C, r, c, eta, norm_mode);
            const bool rleaf = R.left[r] < 0, cleaf = C.left[c] < 0;
            const int8_t st = adm ? 0 : ((rleaf && cleaf) ? 1 : 2);
            o->row.push_back(r);
            o->col.push_back(c);
            o->state.push_back(st);
            o->level.push_back(lev);
            o->key.push_back(fkey[i]);
            o->parent.push_back(fpar[i]);
            if (st == 2) sub.push_back(i);
        }
        base += m;
        if (sub.empty()) break;
        int64_t scale = 1;
        for (int k = 0; k < digits - 1 - lev; ++k) scale *= 4;
        nr.clear(); nc.clear(); nk.clear(); np_.clear();
        for (int a = 0; a < 2; ++a) {
            for (int b = 0; b < 2; ++b) {
                for (int64_t i : sub) {
                    const int64_t r = fr[i], c = fc[i];
                    const bool rs = R.left[r] >= 0, cs = C.left[c] >= 0;
                    const int64_t rk = a == 0 ? (rs ? R.left[r] : r) : (rs ? R.right[r] : -1);
                    const int64_t ck = b == 0 ? (cs ? C.left[c] : c) : (cs ? C.right[c] : -1);
                    if (rk < 0 || ck < 0) continue;
                    const int64_t dig = a * (cs ? 2 : 1) + b;
                    nr.push_back(rk);
                    nc.push_back(ck);
                    nk.push_back(fkey[i] + dig * scale);
                    np_.push_back(base - m + i);
                }
            }
        }
        fr.swap(nr);
        fc.swap(nc);
        fkey.swap(nk);
        fpar.swap(np_);
        ++lev;
    }
    *count = base;
    *handle = o;
    return GC_OK;
}

// Copy the nodes of a gc_block_tree handle into caller arrays of *count
// entries (any pointer may be NULL) and free the handle.
int gc_block_tree_fetch(void* handle, int64_t* row, int64_t* col, int8_t* state, int64_t* level, int64_t* key,
                        int64_t* parent) {
    using namespace gcb;
    BlockTreeOut* o = (BlockTreeOut*)handle;
    if (!o) { set_error(GC_ERR_CONFIG, "gc_block_tree_fetch: null handle"); return GC_ERR_CONFIG; }
    const size_t n = o->row.size();
    if (row) std::copy(o->row.begin(), o->row.end(), row);
    if (col) std::copy(o->col.begin(), o->col.end(), col);
    if (state) std::copy(o->state.begin(), o->state.end(), state);
    if (level) std::copy(o->level.begin(), o->level.end(), level);
    if (key) std::copy(o->key.begin(), o->key.end(), key);
    if (parent) std::copy(o->parent.begin(), o->parent.end(), parent);
    (void)n;
    delete o;
    return GC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The same build on the device, one tree level per call (gc_bt_level): the
// admissibility of every frontier pair (same rounding as above: explicit
// round-to-nearest products and sums, no contraction), its node record at
// out[base + i], and the children of the subdivided pairs written in the
// host routine's order - grouped by child slot q = 2a + b, then by parent -
// through one exclusive scan over the slot-major flags.

namespace gcb {

struct BtTree {
    const double* diam;
    const double* lower;
    const double* upper;
    const int64_t* left;
    const int64_t* right;
};

__device__ __forceinline__ double bt_norm_plain(double a, double b, double c) {
    return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

__device__ __forceinline__ double bt_norm_blas(double x, double y, double z, int mode) {
    if (mode == 0) return sqrt(fma(z, z, fma(y, y, __dmul_rn(x, x))));
    return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// frontier size m and node offset base of this level in meta[0], meta[1]
// (device); the flags are slot-major with stride cap_f (entries past m are
// zero, so the scan orders the children exactly as a stride-m layout would)
__global__ void k_bt_eval(const int64_t* __restrict__ meta, int64_t cap_f, const int64_t* __restrict__ fr,
                          const int64_t* __restrict__ fc, const int64_t* __restrict__ fkey,
                          const int64_t* __restrict__ fpar, int64_t lev, BtTree R, BtTree C, double eta, int mode,
                          int64_t* __restrict__ o_row, int64_t* __restrict__ o_col, int8_t* __restrict__ o_state,
                          int64_t* __restrict__ o_level, int64_t* __restrict__ o_key, int64_t* __restrict__ o_parent,
                          int32_t* __restrict__ flags) {
    const int64_t m = meta[0], base = meta[1];
    if (m == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap_f; i += (int64_t)gridDim.x * blockDim.x) {
        if (i >= m) {
            flags[i] = 0;
            flags[cap_f + i] = 0;
            flags[2 * cap_f + i] = 0;
            flags[3 * cap_f + i] = 0;
            continue;
        }
        const int64_t r = fr[i], c = fc[i];
        const double d = R.diam[r] > C.diam[c] ? R.diam[r] : C.diam[c];
        double g[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double a = __dsub_rn(R.lower[3 * r + k], C.upper[3 * c + k]);
            const double b = __dsub_rn(C.lower[3 * c + k], R.upper[3 * r + k]);
            const double mx = a >= b ? a : b;
            g[k] = mx >= 0.0 ? mx : 0.0;
        }
        const double two_eta = __dmul_rn(2.0, eta);
        const double rhs = __dmul_rn(two_eta, bt_norm_plain(g[0], g[1], g[2]));
        const double big = d > rhs ? d : rhs;
        bool adm;
        if (fabs(__dsub_rn(d, rhs)) <= __dmul_rn(1e-12, big))
            adm = d <= __dmul_rn(two_eta, bt_norm_blas(g[0], g[1], g[2], mode));
        else
            adm = d <= rhs;
        const bool rs = R.left[r] >= 0, cs = C.left[c] >= 0;
        const int8_t st = adm ? 0 : ((!rs && !cs) ? 1 : 2);
        const int64_t id = base + i;
        o_row[id] = r;
        o_col[id] = c;
        o_state[id] = st;
        o_level[id] = lev;
        o_key[id] = fkey[i];
        o_parent[id] = fpar[i];
        const bool sub = st == 2;
        flags[i] = sub;                                   // (a, b) = (0, 0): always present
        flags[cap_f + i] = sub && cs;                     // (0, 1)
        flags[2 * cap_f + i] = sub && rs;                 // (1, 0)
        flags[3 * cap_f + i] = sub && rs && cs;           // (1, 1)
    }
}

// children of the subdivided pairs; the next level's meta (m, base) and
// err bits: 1 frontier capacity, 2 node capacity, 4 key digits exhausted
__global__ void k_bt_children(int64_t* __restrict__ meta, int64_t cap_f, int64_t cap_n, int64_t lev, int32_t digits,
                              const int64_t* __restrict__ fr, const int64_t* __restrict__ fc,
                              const int64_t* __restrict__ fkey, int64_t scale, BtTree R, BtTree C,
                              const int32_t* __restrict__ flags, const int32_t* __restrict__ pos,
                              int64_t* __restrict__ nr, int64_t* __restrict__ nc, int64_t* __restrict__ nk,
                              int64_t* __restrict__ np, int32_t* __restrict__ err) {
    const int64_t m = meta[0], base = meta[1];
    const int64_t total = 4 * cap_f;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t count = m == 0 ? 0 : (int64_t)pos[total - 1] + flags[total - 1];
        int32_t e = 0;
        if (count > cap_f) e |= 1;
        if (base + m + count > cap_n) e |= 2;
        if (count > 0 && lev + 1 >= digits) e |= 4;
        if (e) {
            atomicOr(err, e);
            count = 0;
        }
        meta[2] = count;
        meta[3] = base + m;
    }
    if (m == 0) return;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        if (!flags[t]) continue;
        const int q = (int)(t / cap_f);
        const int64_t i = t - (int64_t)q * cap_f;
        const int64_t p = pos[t];
        if (p >= cap_f) continue;                         // overflow: reported above
        const int a = q >> 1, b = q & 1;
        const int64_t r = fr[i], c = fc[i];
        const bool rs = R.left[r] >= 0, cs = C.left[c] >= 0;
        const int64_t rk = a == 0 ? (rs ? R.left[r] : r) : R.right[r];
        const int64_t ck = b == 0 ? (cs ? C.left[c] : c) : C.right[c];
        const int64_t dig = a * (cs ? 2 : 1) + b;
        nr[p] = rk;
        nc[p] = ck;
        nk[p] = fkey[i] + dig * scale;
        np[p] = base + i;
    }
}

}  // namespace gcb

extern "C" {

// One level of the device block tree without a host read: the level's
// frontier size and node offset in meta[0..1] [dev], the next level's written
// to meta[2..3]; tree arrays [dev] as gc_block_tree; frontier [dev] fr, fc,
// fkey, fpar (capacity cap_f); node records at out_*[base ..] [dev]
// (capacity cap_n); next frontier [dev] nr, nc, nk, np (capacity cap_f);
// flags / pos [dev] 4 cap_f int32 each; err [dev] int32 (1 frontier, 2 node
// capacity, 4 key digits exhausted: the level then ends the tree); temp
// [dev] of gc_bt_level_bytes(cap_f) bytes.  An empty level is a no-op.
int gc_bt_level_bytes(int64_t cap_f, int64_t* bytes) {
    using namespace gcb;
    size_t tb = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr,
                                                  (int)(4 * cap_f));
    if (e != cudaSuccess) return cuda_status(e, "gc_bt_level_bytes");
    *bytes = (int64_t)tb;
    return GC_OK;
}

int gc_bt_level(int64_t* meta, int64_t cap_f, int64_t cap_n, const int64_t* fr, const int64_t* fc,
                const int64_t* fkey, const int64_t* fpar, int64_t lev, int32_t digits, const double* r_diam,
                const double* r_lower, const double* r_upper, const int64_t* r_left, const int64_t* r_right,
                const double* c_diam, const double* c_lower, const double* c_upper, const int64_t* c_left,
                const int64_t* c_right, double eta, int32_t norm_mode, int64_t* o_row, int64_t* o_col,
                int8_t* o_state, int64_t* o_level, int64_t* o_key, int64_t* o_parent, int64_t* nr, int64_t* nc,
                int64_t* nk, int64_t* np, int32_t* flags, int32_t* pos, int32_t* err, void* temp,
                int64_t temp_bytes, void* stream) {
    using namespace gcb;
    if (cap_f <= 0 || 4 * cap_f >= (1LL << 31) || (norm_mode != 0 && norm_mode != 1) || lev >= digits ||
        eta <= 0.0 || !meta || !err) {
        set_error(GC_ERR_CONFIG, "gc_bt_level: bad arguments");
        return GC_ERR_CONFIG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const BtTree R{r_diam, r_lower, r_upper, r_left, r_right};
    const BtTree C{c_diam, c_lower, c_upper, c_left, c_right};
    int64_t grid = (cap_f + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    k_bt_eval<<<(unsigned)grid, 256, 0, st>>>(meta, cap_f, fr, fc, fkey, fpar, lev, R, C, eta, norm_mode, o_row,
                                              o_col, o_state, o_level, o_key, o_parent, flags);
    GC_CHECK_LAUNCH("k_bt_eval");
    size_t tb = (size_t)temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, flags, pos, (int)(4 * cap_f), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_bt_level scan");
    int64_t scale = 1;
    for (int k = 0; k < digits - 1 - lev; ++k) scale *= 4;
    int64_t cgrid = (4 * cap_f + 255) / 256;
    if (cgrid > 148 * 16) cgrid = 148 * 16;
    k_bt_children<<<(unsigned)cgrid, 256, 0, st>>>(meta, cap_f, cap_n, lev, digits, fr, fc, fkey, scale, R, C,
                                                   flags, pos, nr, nc, nk, np, err);
    GC_CHECK_LAUNCH("k_bt_children");
    return GC_OK;
}

}  // extern "C"

namespace gcb {

__global__ void k_bt_leaf_flags(int64_t n, const int8_t* __restrict__ state, char* __restrict__ flag,
                                int64_t* __restrict__ ids) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        flag[i] = state[i] != 2;
        ids[i] = i;
    }
}

__global__ void k_bt_gather_flags(int64_t n, const char* __restrict__ flag, const int64_t* __restrict__ ids,
                                  char* __restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = flag[ids[j]];
}

}  // namespace gcb

extern "C" {

// Leaves of a device block tree in depth-first order (FlatBlockTree's
// leaf_ids / leaf_key): every node sorted by its path key (stable radix;
// a node shares its key only with its first descendants, never with
// another leaf), then the leaves selected in that order.  Scratch [dev]:
// ids, ids_sorted, key_sorted (n int64 each), flag, flag_sorted (n bytes
// each), temp of gc_bt_leaves_bytes(n) bytes; *count [dev] = leaves.
int gc_bt_leaves_bytes(int64_t n, int64_t* bytes) {
    using namespace gcb;
    size_t t1 = 0, t2 = 0;
    cudaError_t e = cub::DeviceSelect::Flagged(nullptr, t1, (const int64_t*)nullptr, (const char*)nullptr,
                                               (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(nullptr, t2, (const int64_t*)nullptr, (int64_t*)nullptr,
                                            (const int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    if (e != cudaSuccess) return cuda_status(e, "gc_bt_leaves_bytes");
    *bytes = (int64_t)(t1 > t2 ? t1 : t2);
    return GC_OK;
}

int gc_bt_leaves(int64_t n, const int8_t* state, const int64_t* key, int64_t* leaf_ids, int64_t* leaf_key,
                 int64_t* count, int64_t* ids, int64_t* ids_sorted, int64_t* key_sorted, char* flag,
                 char* flag_sorted, void* temp, int64_t temp_bytes, void* stream) {
    using namespace gcb;
    if (n <= 0 || n >= (1LL << 31)) { set_error(GC_ERR_CONFIG, "gc_bt_leaves: bad size"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    int64_t grid = (n + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    k_bt_leaf_flags<<<(unsigned)grid, 256, 0, st>>>(n, state, flag, ids);
    GC_CHECK_LAUNCH("k_bt_leaf_flags");
    size_t tb = (size_t)temp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, tb, key, key_sorted, ids, ids_sorted, (int)n, 0, 64, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_bt_leaves sort");
    k_bt_gather_flags<<<(unsigned)grid, 256, 0, st>>>(n, flag, ids_sorted, flag_sorted);
    GC_CHECK_LAUNCH("k_bt_gather_flags");
    tb = (size_t)temp_bytes;
    e = cub::DeviceSelect::Flagged(temp, tb, ids_sorted, flag_sorted, leaf_ids, count, (int)n, st);
    if (e == cudaSuccess) {
        tb = (size_t)temp_bytes;
        e = cub::DeviceSelect::Flagged(temp, tb, key_sorted, flag_sorted, leaf_key, count, (int)n, st);
    }
    if (e != cudaSuccess) return cuda_status(e, "gc_bt_leaves select");
    count_launch(3);
    return GC_OK;
}

}  // extern "C"

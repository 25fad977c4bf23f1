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

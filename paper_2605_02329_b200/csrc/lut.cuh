// lut.cuh — DecodeStepLUT (costmodel.py:61-227) and the decode/prefill cost
// formulas of the ground truth, as device code.
//
// Layout: a compact [nb][ns] grid of f64 sums, f64 means, f64 slopes (np.interp
// slope from each populated column to the next populated column of the same
// row, costmodel.py:153-155 -> numpy arr_interp) and i32 counts, plus a u64
// populated-column mask per row and a u32 populated-row mask.  Means and
// slopes are recomputed for the touched cells at each update (one division per
// affected value), so a lookup costs at most one division (the across-row
// Python-form interpolation, costmodel.py:183-187).
#pragma once
#include "numerics.cuh"

namespace slosim {

struct DLut {
    int nb, ns;
    const int32_t* bb;  // bsz buckets [nb]
    const int32_t* sb;  // seq buckets [ns]
    double* sum;        // [nb*ns]
    double* mean;       // [nb*ns]
    double* slope;      // [nb*ns]
    int32_t* cnt;       // [nb*ns]
    uint64_t* colmask;  // [nb]
    uint32_t rowmask;
};

__device__ __forceinline__ int bisect_left(const int32_t* a, int n, int64_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((int64_t)a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// _bucket_index costmodel.py:99-103: smallest bucket >= value, clamped.
__device__ __forceinline__ int bucket_index(const int32_t* a, int n, int64_t x) {
    int i = bisect_left(a, n, x);
    return i < n - 1 ? i : n - 1;
}

__device__ __forceinline__ uint64_t low_mask64(int j) { return j >= 64 ? ~0ULL : ((1ULL << j) - 1ULL); }

// Recompute the np.interp slope leaving column j of row i (to the next populated column).
__device__ __forceinline__ void lut_fix_slope(DLut& L, int i, int j) {
    uint64_t m = L.colmask[i] & ~low_mask64(j + 1);
    if (m == 0) return;
    int nx = __ffsll((long long)m) - 1;
    int c = i * L.ns;
    L.slope[c + j] = xdiv(xsub(L.mean[c + nx], L.mean[c + j]), xsub((double)L.sb[nx], (double)L.sb[j]));
}

// Single-thread (re)build of row i's means, mask and slopes.
__device__ void lut_build_row(DLut& L, int i) {
    uint64_t m = 0;
    int c = i * L.ns;
    for (int j = 0; j < L.ns; j++) {
        if (L.cnt[c + j] > 0) {
            m |= 1ULL << j;
            L.mean[c + j] = xdiv(L.sum[c + j], (double)L.cnt[c + j]);
        }
    }
    L.colmask[i] = m;
    if (m) L.rowmask |= 1u << i; else L.rowmask &= ~(1u << i);
    for (int j = 0; j < L.ns; j++)
        if ((m >> j) & 1ULL) lut_fix_slope(L, i, j);
}

// np.interp(seq, xs, ys) over the populated columns of row r; j0 = bisect_left(sb, seq).
__device__ __forceinline__ double lut_row_eval(const DLut& L, int r, int64_t seq, int j0) {
    uint64_t m = L.colmask[r];
    int c = r * L.ns;
    int first = __ffsll((long long)m) - 1;
    int last = 63 - __clzll((long long)m);
    if (first == last) return L.mean[c + first];
    if (seq <= (int64_t)L.sb[first]) return L.mean[c + first];
    if (seq >= (int64_t)L.sb[last]) return L.mean[c + last];
    if (j0 < L.ns && (int64_t)L.sb[j0] == seq && ((m >> j0) & 1ULL)) return L.mean[c + j0];
    int jp = 63 - __clzll((long long)(m & low_mask64(j0)));
    // numpy: slope*(x - xp[j]) + fp[j]
    return xadd(xmul(L.slope[c + jp], xsub((double)seq, (double)L.sb[jp])), L.mean[c + jp]);
}

// DecodeStepLUT.lookup costmodel.py:157-187 (bsz, seq >= 1; LUT non-empty).
__device__ __forceinline__ double lut_lookup(const DLut& L, int64_t bsz, int64_t seq) {
    int i = bisect_left(L.bb, L.nb, bsz);
    int j0 = bisect_left(L.sb, L.ns, seq);
    if (i < L.nb && (int64_t)L.bb[i] == bsz && j0 < L.ns && (int64_t)L.sb[j0] == seq && L.cnt[i * L.ns + j0] > 0)
        return L.mean[i * L.ns + j0];
    uint32_t below = L.rowmask & ((1u << i) - 1u);
    uint32_t above = i >= 32 ? 0u : (L.rowmask >> i);
    if (below == 0) return lut_row_eval(L, __ffs((int)L.rowmask) - 1, seq, j0);
    if (above == 0) return lut_row_eval(L, 31 - __clz((int)L.rowmask), seq, j0);
    int rhi = i + __ffs((int)above) - 1;
    if ((int64_t)L.bb[rhi] == bsz) return lut_row_eval(L, rhi, seq, j0);
    int rlo = 31 - __clz((int)below);
    double vlo = lut_row_eval(L, rlo, seq, j0);
    double vhi = lut_row_eval(L, rhi, seq, j0);
    // v_lo + (v_hi - v_lo) * (bsz - b_lo) / (b_hi - b_lo)
    return xadd(vlo, xdiv(xmul(xsub(vhi, vlo), (double)(bsz - L.bb[rlo])), (double)(L.bb[rhi] - L.bb[rlo])));
}

// DecodeStepLUT.update costmodel.py:118-128 (single thread).
__device__ void lut_update(DLut& L, int64_t bsz, int64_t max_seq, int64_t obs) {
    int i = bucket_index(L.bb, L.nb, bsz), j = bucket_index(L.sb, L.ns, max_seq);
    int c = i * L.ns + j;
    bool fresh = L.cnt[c] == 0;
    L.sum[c] = xadd(L.sum[c], (double)obs);
    L.cnt[c] += 1;
    if (fresh) { lut_build_row(L, i); return; }
    L.mean[c] = xdiv(L.sum[c], (double)L.cnt[c]);
    lut_fix_slope(L, i, j);
    uint64_t prev = L.colmask[i] & low_mask64(j);
    if (prev) lut_fix_slope(L, i, 63 - __clzll((long long)prev));
}

// _interp_clamped costmodel.py:32-47 (Python form y0 + (y1-y0)*(x-x0)/(x1-x0)).
__device__ __forceinline__ double interp_clamped(int n, const int64_t* px, const double* py, int64_t x) {
    if (x <= px[0]) return py[0];
    if (x >= px[n - 1]) return py[n - 1];
    int k = 0;
    while (k + 1 < n && px[k + 1] <= x) k++;
    double y0 = py[k], y1 = py[k + 1];
    return xadd(y0, xdiv(xmul(xsub(y1, y0), (double)(x - px[k])), (double)(px[k + 1] - px[k])));
}

// decode_step_formula costmodel.py:50-58.
__device__ __forceinline__ double decode_formula(int n, const int64_t* bx, const double* by, double gamma,
                                                 int64_t bsz, int64_t seq) {
    return xmul(interp_clamped(n, bx, by, seq), xadd(1.0, xmul(gamma, (double)(bsz - 1))));
}

// _GroundTruth._curve_at engine.py:161-173 (integer points; int + int*int/int).
__device__ __forceinline__ double curve_at(int n, const int64_t* x, const int64_t* y, int64_t tokens) {
    if (tokens >= x[n - 1]) {
        int64_t x0 = x[n - 2], y0 = y[n - 2], x1 = x[n - 1], y1 = y[n - 1];
        return xadd((double)y1, idiv_prod(y1 - y0, tokens - x1, x1 - x0));
    }
    int k = 0;
    while (tokens > x[k + 1]) k++;
    int64_t x0 = x[k], y0 = y[k], x1 = x[k + 1], y1 = y[k + 1];
    return xadd((double)y0, idiv_prod(y1 - y0, tokens - x0, x1 - x0));
}

}  // namespace slosim

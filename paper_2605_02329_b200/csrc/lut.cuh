// lut.cuh — DecodeStepLUT (costmodel.py:61-227) and the ground-truth cost
// formulas (costmodel.py:32-58, engine.py:161-192) as device code.
//
// One LUT is one LutMem block (reached through a single pointer, so it costs
// two registers): compact [nb][ns] grids of f64 sums, means and np.interp
// slopes (slope from each populated column to the next populated column of
// its row), i32 counts, a u64 populated-column mask per row, a populated-row
// mask, copies of the bucket arrays and two direct-index tables that replace
// the bisections of the reference (bisect_left over bsz for b <= 256 and a
// 256-entry coarse table over seq_len refined by <= a couple of steps).
//
// Fast path: once every cell is populated (true from the start for
// synthesized profiles with prior_weight > 0, and forever after because
// counts only grow) a lookup is   row selection(bsz) x column selection(seq)
// -> slope*dx + mean per row, plus one division for the across-row Python-form
// interpolation.  The column selection of a candidate is computed once per
// decode step and reused across the greedy scan's rounds.
#pragma once
#include "numerics.cuh"

namespace slosim {

#define LUT_CELLS (SLOSIM_MAX_BSZ_BUCKETS * SLOSIM_MAX_SEQ_BUCKETS)

struct LutMem {
    double sum[LUT_CELLS];
    double mean[LUT_CELLS];
    double slope[LUT_CELLS];
    int32_t cnt[LUT_CELLS];
    uint64_t colmask[SLOSIM_MAX_BSZ_BUCKETS];
    int32_t bb[SLOSIM_MAX_BSZ_BUCKETS];
    int32_t sb[SLOSIM_MAX_SEQ_BUCKETS];
    int32_t nb, ns, sshift, full;
    uint32_t rowmask;
    int32_t populated;
    int32_t geo;  // 1: bsz buckets 2^0..2^(nb-1) and seq buckets (j+1) << wsh (index math, no tables)
    int32_t wsh;
    int32_t bad;  // 1: the profile is malformed (build_profile_tables)
    uint8_t bidx[264];  // bidx[b] = bisect_left(bb, b), b <= 256
    uint8_t sidx[264];  // sidx[q] = bisect_left(sb, q << sshift), q <= 256
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

__device__ __noinline__ int bisect_left_call(const int32_t* a, int n, int64_t x) { return bisect_left(a, n, x); }

__device__ __forceinline__ int lut_bidx(const LutMem* L, int64_t b) {
    return (b >= 0 && b <= 256) ? (int)L->bidx[b] : bisect_left_call(L->bb, L->nb, b);
}

__device__ __forceinline__ int lut_sidx(const LutMem* L, int64_t s) {
    int64_t q = s >> L->sshift;
    if (q < 0 || q > 256) return bisect_left_call(L->sb, L->ns, s);
    int j = L->sidx[q];
    while (j < L->ns && (int64_t)L->sb[j] < s) j++;
    return j;
}

__device__ __forceinline__ uint64_t low_mask64(int j) { return j >= 64 ? ~0ULL : ((1ULL << j) - 1ULL); }

// Recompute the slope leaving column j of row i (to the next populated column).
__device__ __forceinline__ void lut_fix_slope(LutMem* L, int i, int j) {
    uint64_t m = L->colmask[i] & ~low_mask64(j + 1);
    int c = i * L->ns;
    if (m == 0) { L->slope[c + j] = 0.0; return; }
    int nx = __ffsll((long long)m) - 1;
    L->slope[c + j] = xdiv(xsub(L->mean[c + nx], L->mean[c + j]), xsub((double)L->sb[nx], (double)L->sb[j]));
}

// Single-thread (re)build of row i's means, mask and slopes.
__device__ __noinline__ void lut_build_row(LutMem* L, int i) {
    uint64_t m = 0;
    int c = i * L->ns;
    for (int j = 0; j < L->ns; j++) {
        if (L->cnt[c + j] > 0) {
            m |= 1ULL << j;
            L->mean[c + j] = xdiv(L->sum[c + j], (double)L->cnt[c + j]);
        } else {
            L->mean[c + j] = 0.0;
        }
        L->slope[c + j] = 0.0;
    }
    L->colmask[i] = m;
    for (int j = 0; j < L->ns; j++)
        if ((m >> j) & 1ULL) lut_fix_slope(L, i, j);
}

// Warp-cooperative build of a LutMem from a 16x64-framed (sums, counts) pair.
__device__ void lut_build(LutMem* L, int nb, int ns, const int32_t* bb, const int32_t* sb, const double* fsums,
                          const int32_t* fcounts, int lane) {
    for (int c = lane; c < nb * ns; c += 32) {
        int i = c / ns, j = c % ns;
        L->sum[c] = fsums[i * SLOSIM_MAX_SEQ_BUCKETS + j];
        L->cnt[c] = fcounts[i * SLOSIM_MAX_SEQ_BUCKETS + j];
    }
    if (lane < nb) L->bb[lane] = bb[lane];
    for (int j = lane; j < ns; j += 32) L->sb[j] = sb[j];
    int sshift = 0;
    while (((int64_t)256 << sshift) < (int64_t)sb[ns - 1]) sshift++;
    if (lane == 0) { L->nb = nb; L->ns = ns; L->sshift = sshift; }  // read by lut_build_row below
    __syncwarp();
    for (int q = lane; q < 264; q += 32) {
        L->bidx[q] = (uint8_t)bisect_left(bb, nb, q);
        L->sidx[q] = (uint8_t)bisect_left(sb, ns, (int64_t)q << sshift);
    }
    if (lane < nb) lut_build_row(L, lane);
    __syncwarp();
    bool pop = lane < nb && L->colmask[lane] != 0;
    uint32_t rm = __ballot_sync(0xffffffffu, pop);
    int cells = 0;
    for (int c = lane; c < nb * ns; c += 32) cells += L->cnt[c] > 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
    int wsh = 0;
    while (wsh < 30 && (1 << wsh) < sb[0]) wsh++;
    bool geo = nb <= 16 && (1 << wsh) == sb[0];
    for (int i = 0; i < nb; i++) geo = geo && bb[i] == (1 << i);
    for (int j = 0; j < ns; j++) geo = geo && (int64_t)sb[j] == ((int64_t)(j + 1) << wsh);
    if (lane == 0) {
        L->rowmask = rm;
        L->populated = cells;
        L->full = cells == nb * ns;
        L->geo = geo ? 1 : 0;
        L->wsh = wsh;
        L->bad = 0;
    }
    __syncwarp();
}

// Copy of a built LutMem (only the live part of the frame).
__device__ void lut_copy(LutMem* dst, const LutMem* src, int lane) {
    int K = src->nb * src->ns;
#pragma unroll 1
    for (int c = lane; c < K; c += 32) {
        dst->sum[c] = src->sum[c]; dst->mean[c] = src->mean[c]; dst->slope[c] = src->slope[c]; dst->cnt[c] = src->cnt[c];
    }
    if (lane < src->nb) { dst->colmask[lane] = src->colmask[lane]; dst->bb[lane] = src->bb[lane]; }
    for (int j = lane; j < src->ns; j += 32) dst->sb[j] = src->sb[j];
    const uint32_t* s32 = (const uint32_t*)src->bidx;
    uint32_t* d32 = (uint32_t*)dst->bidx;
    for (int k = lane; k < 2 * 264 / 4; k += 32) d32[k] = s32[k];
    if (lane == 0) {
        dst->nb = src->nb; dst->ns = src->ns; dst->sshift = src->sshift; dst->full = src->full;
        dst->rowmask = src->rowmask; dst->populated = src->populated;
        dst->geo = src->geo; dst->wsh = src->wsh;
    }
    __syncwarp();
}

// ---- full-grid fast path ----------------------------------------------------
// G = true: the power-of-two geometry (L->geo; the reference's default buckets
// costmodel.py:26-27 are of this shape).  Bucket indices are then integer
// arithmetic, and every divisor of the interpolations (b_hi - b_lo = 2^k across
// rows, the seq bucket width 2^wsh along a row) is a power of two, so the
// correctly rounded quotient is the exact product with 2^-k: same bits, one
// DMUL instead of a DDIV.
struct ColSel { int c; double dx; };   // value of a row = slope[row][c]*dx + mean[row][c]
struct RowSel { int r1, r2; int64_t num, den; double inv; };  // r2 < 0: single row r1; inv = 1/den (G)

__device__ __forceinline__ double pow2_neg(int k) { return __longlong_as_double((long long)(1023 - k) << 52); }

// bisect_left over the geometry: smallest i with 2^i >= b (b >= 1), smallest j with (j+1) << wsh >= s (s >= 1)
__device__ __forceinline__ int geo_bidx(int64_t b) { return b <= 1 ? 0 : 64 - __clzll((long long)(b - 1)); }
__device__ __forceinline__ int geo_sidx(const LutMem* L, int64_t s) {
    return (int)(((s + ((int64_t)1 << L->wsh) - 1) >> L->wsh) - 1);
}

// np.interp column selection (numpy arr_interp) for a fully populated row.
template <bool G = false>
__device__ __forceinline__ ColSel lut_col(const LutMem* L, int64_t seq) {
    int ns = L->ns;
    if (G) {
        // c = floor(seq / W) - 1 and dx = seq mod W inside the grid (dx = 0 at a node), clamped outside
        const int w = L->wsh;
        int64_t c = (seq >> w) - 1;
        bool in = seq > ((int64_t)1 << w) && c < ns - 1;
        return ColSel{in ? (int)c : (seq <= ((int64_t)1 << w) ? 0 : ns - 1), in ? (double)(seq & (((int64_t)1 << w) - 1)) : 0.0};
    }
    if (seq <= (int64_t)L->sb[0]) return ColSel{0, 0.0};
    if (seq >= (int64_t)L->sb[ns - 1]) return ColSel{ns - 1, 0.0};
    int j0 = lut_sidx(L, seq);
    if ((int64_t)L->sb[j0] == seq) return ColSel{j0, 0.0};
    return ColSel{j0 - 1, xsub((double)seq, (double)L->sb[j0 - 1])};
}

// Row selection of lookup() (costmodel.py:175-187) when every row is populated.
template <bool G = false>
__device__ __forceinline__ RowSel lut_rows(const LutMem* L, int64_t bsz) {
    if (G) {
        int i = geo_bidx(bsz);
        if (i == 0) return RowSel{0, -1, 0, 1, 1.0};
        if (i >= L->nb) return RowSel{L->nb - 1, -1, 0, 1, 1.0};
        if (((int64_t)1 << i) == bsz) return RowSel{i, -1, 0, 1, 1.0};
        return RowSel{i - 1, i, bsz - ((int64_t)1 << (i - 1)), (int64_t)1 << (i - 1), pow2_neg(i - 1)};
    }
    int i = lut_bidx(L, bsz);
    if (i == 0) return RowSel{0, -1, 0, 1, 1.0};
    if (i == L->nb) return RowSel{L->nb - 1, -1, 0, 1, 1.0};
    if ((int64_t)L->bb[i] == bsz) return RowSel{i, -1, 0, 1, 1.0};
    return RowSel{i - 1, i, bsz - L->bb[i - 1], (int64_t)L->bb[i] - L->bb[i - 1], 1.0};
}

// Branch-free row selection for per-lane batch sizes (speculative scan).
template <bool G = false>
__device__ __forceinline__ RowSel lut_rows_nb(const LutMem* L, int64_t bsz) {
    int nb = L->nb;
    RowSel rs;
    if (G) {
        int i = geo_bidx(bsz);
        bool single = (i == 0) | (i >= nb) | (((int64_t)1 << i) == bsz);
        int lo = i >= nb ? nb - 1 : (i == 0 ? 0 : i - 1);
        rs.r1 = single ? (i >= nb ? nb - 1 : i) : lo;
        rs.r2 = single ? -1 : i;
        rs.num = single ? 0 : bsz - ((int64_t)1 << lo);
        rs.den = single ? 1 : (int64_t)1 << lo;
        rs.inv = pow2_neg(single ? 0 : lo);
        return rs;
    }
    int i = lut_bidx(L, bsz);
    int ic = i < nb ? i : nb - 1;
    int64_t bi = L->bb[ic];
    bool single = (i == 0) | (i == nb) | (bi == bsz);
    int r1 = i == 0 ? 0 : (i == nb ? nb - 1 : (bi == bsz ? i : i - 1));
    int64_t blo = L->bb[r1];
    rs.r1 = r1;
    rs.r2 = single ? -1 : i;
    rs.num = single ? 0 : bsz - blo;
    rs.den = single ? 1 : bi - blo;
    rs.inv = 1.0;
    return rs;
}

template <bool G = false>
__device__ __forceinline__ double lut_eval(const LutMem* L, const RowSel& rs, const ColSel& cs) {
    int ns = L->ns;
    int k1 = rs.r1 * ns + cs.c;
    double v1 = xadd(xmul(L->slope[k1], cs.dx), L->mean[k1]);
    if (rs.r2 < 0) return v1;
    int k2 = rs.r2 * ns + cs.c;
    double v2 = xadd(xmul(L->slope[k2], cs.dx), L->mean[k2]);
    // v_lo + (v_hi - v_lo) * (bsz - b_lo) / (b_hi - b_lo)
    // (power-of-two weights: RN(RN(d * num) * 2^-lo) = RN(d * (num * 2^-lo)), one multiply)
    if (G) return xadd(v1, xmul(xsub(v2, v1), (double)rs.num * rs.inv));
    return xadd(v1, xdiv(xmul(xsub(v2, v1), (double)rs.num), (double)rs.den));
}

// ---- power-of-two geometry, hot-loop forms ----------------------------------
// The same arithmetic as lut_col/lut_rows_nb/lut_eval/lut_update_warp<true>,
// with the instance-invariant geometry held in registers (Geo), 32-bit
// indices, both rows always loaded (no branch on a single row) and the cell
// update written branch-free with predicated stores.
struct Geo { int nb, ns, wsh; };
__device__ __forceinline__ Geo geo_of(const LutMem* L) { return Geo{L->nb, L->ns, L->wsh}; }
__device__ __forceinline__ int gbidx(int b) { return b <= 1 ? 0 : 32 - __clz(b - 1); }

__device__ __forceinline__ ColSel gcol(const Geo& g, int seq) {
    const int w = 1 << g.wsh;
    const int c = (seq >> g.wsh) - 1;
    const bool in = seq > w && c < g.ns - 1;
    return ColSel{in ? c : (seq <= w ? 0 : g.ns - 1), in ? (double)(seq & (w - 1)) : 0.0};
}

__device__ __forceinline__ RowSel grows(const Geo& g, int bsz) {
    const int i = gbidx(bsz);
    const bool single = (i == 0) | (i >= g.nb) | ((1u << i) == (unsigned)bsz);
    const int lo = i >= g.nb ? g.nb - 1 : (i == 0 ? 0 : i - 1);
    RowSel rs;
    rs.r1 = single ? (i >= g.nb ? g.nb - 1 : i) : lo;
    rs.r2 = single ? -1 : i;
    rs.num = single ? 0 : bsz - (1 << lo);
    rs.den = single ? 1 : (1 << lo);
    rs.inv = pow2_neg(single ? 0 : lo);
    return rs;
}

__device__ __forceinline__ double geval(const LutMem* L, const Geo& g, const RowSel& rs, const ColSel& cs) {
    const int k1 = rs.r1 * g.ns + cs.c;
    const int k2 = (rs.r2 < 0 ? rs.r1 : rs.r2) * g.ns + cs.c;
    const double v1 = xadd(xmul(L->slope[k1], cs.dx), L->mean[k1]);
    const double v2 = xadd(xmul(L->slope[k2], cs.dx), L->mean[k2]);
    const double r = xadd(v1, xmul(xsub(v2, v1), (double)rs.num * rs.inv));
    return rs.r2 < 0 ? v1 : r;
}

// Row selection of batch sizes 1..32 (the register-mode scan) as a per-warp
// table: rows r1, r2 (r2 = r1 for a single row) and the Python-form weight
// num * 2^-lo.  A single row then evaluates as v1 + (v1 - v1) * 0 = v1 exactly
// (LUT means are positive), so the evaluation needs no select.
struct RowP { int16_t r1, r2; int32_t num; double wgt; };  // wgt = num * 2^-lo, exact
__device__ __forceinline__ RowP rowp_of(const Geo& g, int bsz) {
    const RowSel rs = grows(g, bsz);
    return RowP{(int16_t)rs.r1, (int16_t)(rs.r2 < 0 ? rs.r1 : rs.r2), (int32_t)rs.num, (double)rs.num * rs.inv};
}
__device__ __forceinline__ double geval_p(const LutMem* L, const Geo& g, const RowP& rp, const ColSel& cs) {
    const int k1 = rp.r1 * g.ns + cs.c, k2 = rp.r2 * g.ns + cs.c;
    const double v1 = xadd(xmul(L->slope[k1], cs.dx), L->mean[k1]);
    const double v2 = xadd(xmul(L->slope[k2], cs.dx), L->mean[k2]);
    return xadd(v1, xmul(xsub(v2, v1), rp.wgt));
}

#ifdef __CUDACC__
__device__ __forceinline__ void st_if(bool p, double* a, double v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.f64 [%1], %2;\n\t}" ::"r"((unsigned)p), "l"(a),
                 "d"(v) : "memory");
}
__device__ __forceinline__ void st_if(bool p, int32_t* a, int32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.s32 [%1], %2;\n\t}" ::"r"((unsigned)p), "l"(a),
                 "r"(v) : "memory");
}
#else  // host test harness (tools/lane_host): plain predicated stores
inline void st_if(bool p, double* a, double v) { if (p) *a = v; }
inline void st_if(bool p, int32_t* a, int32_t v) { if (p) *a = v; }
#endif

// DecodeStepLUT.update (costmodel.py:118-128) on a full power-of-two grid:
// lane 0 writes the cell, lane 1 the slope out of it, lane 2 the slope into it.
// The neighbour mean is loaded by every lane (cells c-1 and c+1 always lie
// inside the LutMem block) and only the stores are predicated.
__device__ __forceinline__ void gupdate(LutMem* L, const Geo& g, int bsz, int max_seq, int64_t obs, int lane,
                                        int32_t add = 1) {
    const int i = min(gbidx(bsz), g.nb - 1);
    const int j = min(((max_seq + (1 << g.wsh) - 1) >> g.wsh) - 1, g.ns - 1);
    const int c = i * g.ns + j;
    const double sum = xadd(L->sum[c], (double)obs);
    const int32_t cnt = L->cnt[c] + add;
    const double mean = xdiv(sum, (double)cnt);
    const bool right = lane == 1 && j + 1 < g.ns, left = lane == 2 && j > 0;
    const double mn = L->mean[lane == 1 ? c + 1 : c - 1];
    const double ma = right ? mean : mn, mb = right ? mn : mean;
    st_if(lane == 0, &L->sum[c], sum);
    st_if(lane == 0, &L->cnt[c], cnt);
    st_if(lane == 0, &L->mean[c], mean);
    st_if(right || left, &L->slope[right ? c : c - 1], xmul(xsub(mb, ma), pow2_neg(g.wsh)));
}

// ---- general path -----------------------------------------------------------
// np.interp(seq, xs, ys) over the populated columns of row r; j0 = bisect_left(sb, seq).
__device__ __forceinline__ double lut_row_eval(const LutMem* L, int r, int64_t seq, int j0) {
    uint64_t m = L->colmask[r];
    int c = r * L->ns;
    int first = __ffsll((long long)m) - 1;
    int last = 63 - __clzll((long long)m);
    if (first == last) return L->mean[c + first];
    if (seq <= (int64_t)L->sb[first]) return L->mean[c + first];
    if (seq >= (int64_t)L->sb[last]) return L->mean[c + last];
    if (j0 < L->ns && (int64_t)L->sb[j0] == seq && ((m >> j0) & 1ULL)) return L->mean[c + j0];
    int jp = 63 - __clzll((long long)(m & low_mask64(j0)));
    return xadd(xmul(L->slope[c + jp], xsub((double)seq, (double)L->sb[jp])), L->mean[c + jp]);
}

// DecodeStepLUT.lookup costmodel.py:157-187, general path (some cells unpopulated).
__device__ __noinline__ double lut_lookup_general(const LutMem* L, int64_t bsz, int64_t seq) {
    int i = lut_bidx(L, bsz);
    int j0 = lut_sidx(L, seq);
    int nb = L->nb, ns = L->ns;
    if (i < nb && (int64_t)L->bb[i] == bsz && j0 < ns && (int64_t)L->sb[j0] == seq && L->cnt[i * ns + j0] > 0)
        return L->mean[i * ns + j0];
    uint32_t rowmask = L->rowmask;
    uint32_t below = rowmask & ((1u << i) - 1u);
    uint32_t above = i >= 32 ? 0u : (rowmask >> i);
    if (below == 0) return lut_row_eval(L, __ffs((int)rowmask) - 1, seq, j0);
    if (above == 0) return lut_row_eval(L, 31 - __clz((int)rowmask), seq, j0);
    int rhi = i + __ffs((int)above) - 1;
    if ((int64_t)L->bb[rhi] == bsz) return lut_row_eval(L, rhi, seq, j0);
    int rlo = 31 - __clz((int)below);
    double vlo = lut_row_eval(L, rlo, seq, j0);
    double vhi = lut_row_eval(L, rhi, seq, j0);
    return xadd(vlo, xdiv(xmul(xsub(vhi, vlo), (double)(bsz - L->bb[rlo])), (double)(L->bb[rhi] - L->bb[rlo])));
}

// DecodeStepLUT.lookup costmodel.py:157-187 (bsz, seq >= 1; LUT non-empty).
__device__ __forceinline__ double lut_lookup(const LutMem* L, int64_t bsz, int64_t seq) {
    if (L->full) return lut_eval(L, lut_rows(L, bsz), lut_col(L, seq));
    return lut_lookup_general(L, bsz, seq);
}

// DecodeStepLUT.update costmodel.py:118-128 (single thread; caller syncs the warp).
__device__ __noinline__ void lut_update(LutMem* L, int64_t bsz, int64_t max_seq, int64_t obs) {
    // _bucket_index: smallest bucket >= key, clamped to the last (table lookups)
    int i = lut_bidx(L, bsz), j = lut_sidx(L, max_seq);
    i = i < L->nb - 1 ? i : L->nb - 1;
    j = j < L->ns - 1 ? j : L->ns - 1;
    int c = i * L->ns + j;
    bool fresh = L->cnt[c] == 0;
    L->sum[c] = xadd(L->sum[c], (double)obs);
    L->cnt[c] += 1;
    if (fresh) {
        lut_build_row(L, i);
        L->rowmask |= 1u << i;
        L->populated += 1;
        L->full = L->populated == L->nb * L->ns;
        return;
    }
    L->mean[c] = xdiv(L->sum[c], (double)L->cnt[c]);
    lut_fix_slope(L, i, j);
    uint64_t prev = L->colmask[i] & low_mask64(j);
    if (prev) lut_fix_slope(L, i, 63 - __clzll((long long)prev));
}

// Warp form of lut_update: on a fully populated grid lanes 0-2 compute the new
// cell mean and the np.interp slopes into and out of the cell concurrently
// (neighbouring columns are the populated neighbours); otherwise lane 0 runs
// the general update.
template <bool G = false>
__device__ __forceinline__ void lut_update_warp(LutMem* L, int64_t bsz, int64_t max_seq, int64_t obs, int lane,
                                                int32_t add = 1) {
    if (!L->full) {
        if (lane == 0) lut_update(L, bsz, max_seq, obs);
        return;
    }
    const int nb = L->nb, ns = L->ns;
    int i = G ? geo_bidx(bsz) : lut_bidx(L, bsz), j = G ? geo_sidx(L, max_seq) : lut_sidx(L, max_seq);
    i = i < nb - 1 ? i : nb - 1;
    j = j < ns - 1 ? j : ns - 1;
    const int c = i * ns + j;
    double sum = xadd(L->sum[c], (double)obs);
    int32_t cnt = L->cnt[c] + add;
    double mean = xdiv(sum, (double)cnt);
    // lane 0: the cell; lane 1: slope (j -> j+1); lane 2: slope (j-1 -> j)
    if (lane == 0) { L->sum[c] = sum; L->cnt[c] = cnt; L->mean[c] = mean; }
    bool right = lane == 1 && j + 1 < ns, left = lane == 2 && j > 0;
    if (right || left) {
        int a = right ? j : j - 1;
        double ma = right ? mean : L->mean[c - 1];
        double mb = right ? L->mean[c + 1] : mean;
        L->slope[i * ns + a] = G ? xmul(xsub(mb, ma), pow2_neg(L->wsh))
                                 : xdiv(xsub(mb, ma), xsub((double)L->sb[a + 1], (double)L->sb[a]));
    }
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

// decode_step_formula for the (common) one- or two-anchor base curve, with
// the anchors staged once per instance (shared memory in the engine): the same
// expression as interp_clamped + decode_formula, without the anchor search.
struct GtLine { double y0, y1, dy, dx, gamma; int64_t x0, x1; };
__device__ __forceinline__ bool gt_line_make(int n, const int64_t* bx, const double* by, double gamma, GtLine& k) {
    if (n < 1 || n > 2) return false;
    k.x0 = bx[0]; k.x1 = bx[n - 1]; k.y0 = by[0]; k.y1 = by[n - 1];
    k.dy = xsub(k.y1, k.y0);
    k.dx = (double)(k.x1 - k.x0);
    k.gamma = gamma;
    return true;
}
__device__ __forceinline__ double gt_line_eval(const GtLine& k, int64_t bsz, int64_t seq) {
#ifdef SLOSIM_GT_BRANCH
    double base = seq <= k.x0 ? k.y0 : k.y1;
    if (seq > k.x0 && seq < k.x1) base = xadd(k.y0, xdiv(xmul(k.dy, (double)(seq - k.x0)), k.dx));
#else
    const double mid = xadd(k.y0, xdiv(xmul(k.dy, (double)(seq - k.x0)), k.dx));
    const double base = seq <= k.x0 ? k.y0 : (seq >= k.x1 ? k.y1 : mid);
#endif
    return xmul(base, xadd(1.0, xmul(k.gamma, (double)(bsz - 1))));
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

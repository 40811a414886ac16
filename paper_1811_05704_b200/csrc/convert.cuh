// Device-side construction of the solve-phase matrix formats
// from a CSR copy on the device: the same arrays amgb.cu's host converters
// (to_sell, tma_cols) build -- SELL-32 slices (entry k of row 32 s + r at
// sptr[s] + 32 k + r, padding = the row's last column with value 0), and for
// the TMA format the per-slice column-offset dictionary and the tile-aligned
// column array.  One thread per slice / tile / row; integer work plus copies
// of values, so the result is bitwise the host converter's
// (tests/test_gpu_setup.py compares solves bitwise).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace amgb {

constexpr int kDictW = 16;  // dictionary slices have at most kDictW offsets

#define CV_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// sw[s + 1] = 32 * (longest row of slice s)
__global__ void cv_slice_width(int64_t nrows, int64_t nslices, const int64_t* ptr, int64_t* sw) {
    CV_LOOP(s, nslices) {
        int64_t w = 0;
        const int64_t r1 = (s + 1) * 32 < nrows ? (s + 1) * 32 : nrows;
        for (int64_t r = s * 32; r < r1; ++r) w = ptr[r + 1] - ptr[r] > w ? ptr[r + 1] - ptr[r] : w;
        sw[s + 1] = 32 * w;
        if (s == 0) sw[0] = 0;
    }
}

// dictionary of slice s (amgb.cu tma_cols): the sorted distinct offsets col - row
// of its 32 rows if there are exactly w of them (w = slice width <= kDictW),
// every row + offset is a valid column and every row's columns are ascending
// (the local matrices of a partition keep the global entry order, so a row whose
// first entry is a ghost is not); ulen[s] = w, else 0
__global__ void cv_dict(int64_t nrows, int64_t ncols, int64_t nslices, const int64_t* ptr, const int32_t* col,
                        const int64_t* sptr, int32_t* U, int32_t* ulen) {
    CV_LOOP(s, nslices) {
        ulen[s] = 0;
        const int64_t w = (sptr[s + 1] - sptr[s]) / 32;
        const int64_t r0 = s * 32, r1 = r0 + 32;
        if (w == 0 || w > kDictW || r1 > nrows) continue;
        int64_t list[kDictW];
        int m = 0;
        bool ok = true;
        for (int64_t r = r0; r < r1 && ok; ++r)
            for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
                if (e > ptr[r] && col[e] <= col[e - 1]) {  // the value layout needs ascending columns
                    ok = false;
                    break;
                }
                const int64_t off = (int64_t)col[e] - r;
                int lo = 0, hi = m;
                while (lo < hi) {
                    const int mid = (lo + hi) / 2;
                    if (list[mid] < off) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < m && list[lo] == off) continue;
                if (m == w) {
                    ok = false;
                    break;
                }
                for (int t = m; t > lo; --t) list[t] = list[t - 1];
                list[lo] = off;
                ++m;
            }
        if (!ok || m != w) continue;
        if (r0 + list[0] < 0 || (r1 - 1) + list[m - 1] >= ncols) continue;
        for (int k = 0; k < m; ++k) U[s * kDictW + k] = (int32_t)list[k];
        ulen[s] = m;
    }
}

// per tile of 8 slices: its column ints (dictionary: w, explicit: 32 w),
// rounded up to 4 (16-byte aligned tiles); tc[t + 1]
__global__ void cv_tile_cols(int64_t nslices, int64_t ntiles, const int64_t* sptr, const int32_t* ulen, int64_t* tc) {
    CV_LOOP(t, ntiles) {
        int64_t c = 0;
        const int64_t s1 = (t + 1) * 8 < nslices ? (t + 1) * 8 : nslices;
        for (int64_t s = t * 8; s < s1; ++s) {
            const int64_t w = (sptr[s + 1] - sptr[s]) / 32;
            c += ulen[s] ? w : 32 * w;
        }
        tc[t + 1] = (c + 3) & ~int64_t(3);
        if (t == 0) tc[0] = 0;
    }
}

// cptr[s] from the tile starts; also per-tile stage size (max of entries and
// column ints) and the per-slice index bytes the format needs
__global__ void cv_cptr(int64_t nslices, int64_t ntiles, const int64_t* ptr, int64_t nrows, const int64_t* sptr,
                        const int32_t* ulen, const int64_t* tstart, int64_t* cptr, int64_t* tile_ent,
                        int64_t* idx_bytes) {
    CV_LOOP(t, ntiles) {
        int64_t cur = tstart[t];
        const int64_t s1 = (t + 1) * 8 < nslices ? (t + 1) * 8 : nslices;
        int64_t ib = 0;
        for (int64_t s = t * 8; s < s1; ++s) {
            cptr[s] = cur;
            const int64_t w = (sptr[s + 1] - sptr[s]) / 32;
            if (ulen[s]) {
                cur += w;
                ib += 4 * w;
            } else {
                cur += 32 * w;
                const int64_t r0 = s * 32, r1 = r0 + 32 < nrows ? r0 + 32 : nrows;
                ib += 4 * (ptr[r1] - ptr[r0]);
            }
        }
        if (t == ntiles - 1) cptr[nslices] = tstart[ntiles];
        const int64_t ents = sptr[s1] - sptr[t * 8], cols = tstart[t + 1] - tstart[t];
        tile_ent[t] = ents > cols ? ents : cols;
        idx_bytes[t] = ib;
    }
}

// one thread per (padded) row: the row's slice entries.  Explicit slices: the
// row's entries then padding (last column, value 0) -- into scol (SELL) and/or
// tcol (TMA: at cptr[s] + 32 k + lane).  Dictionary slices: values at the
// dictionary positions, zero where the row lacks an offset; lane 0 writes the
// dictionary to tcol.
__global__ void cv_fill(int64_t nrows, int64_t nslices, const int64_t* ptr, const int32_t* col, const double* val,
                        const int64_t* sptr, const int32_t* ulen, const int32_t* U, const int64_t* cptr, int32_t* scol,
                        int32_t* tcol, double* sval) {
    CV_LOOP(r, nslices * 32) {
        const int64_t s = r >> 5;
        const int lane = (int)(r & 31);
        const int64_t base = sptr[s] + lane;
        const int64_t w = (sptr[s + 1] - sptr[s]) / 32;
        const bool dict = ulen && ulen[s] > 0;
        const int64_t b = r < nrows ? ptr[r] : 0, e = r < nrows ? ptr[r + 1] : 0;
        if (dict) {
            const int32_t* u = U + s * kDictW;
            int64_t k = 0;
            for (int64_t q = b; q < e; ++q) {
                const int64_t off = (int64_t)col[q] - r;
                for (; u[k] != off; ++k) sval[base + 32 * k] = 0.0;
                sval[base + 32 * k] = val[q];
                ++k;
            }
            for (; k < w; ++k) sval[base + 32 * k] = 0.0;
            if (lane == 0)
                for (int64_t q = 0; q < w; ++q) tcol[cptr[s] + q] = u[q];
        } else {
            const int32_t last = e > b ? col[e - 1] : 0;
            for (int64_t k = 0; k < w; ++k) {
                const bool in = b + k < e;
                const int32_t c = in ? col[b + k] : last;
                sval[base + 32 * k] = in ? val[b + k] : 0.0;
                if (scol) scol[base + 32 * k] = c;
                if (tcol) tcol[cptr[s] + 32 * k + lane] = c;
            }
        }
    }
}

__global__ void cv_ptr32(int64_t n, const int64_t* p, int32_t* q) {
    CV_LOOP(i, n) q[i] = (int32_t)p[i];
}

__global__ void cv_to_f32(int64_t n, const double* v, float* f) {
    CV_LOOP(i, n) f[i] = (float)v[i];
}

}  // namespace amgb

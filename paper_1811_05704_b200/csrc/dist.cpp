// Row partition and halo plans (see dist.hpp).
#include "dist.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

namespace amgb {

int first_replicated_level(const HostHierarchy& H, int nranks, int64_t gather_below) {
    const int L = (int)H.levels.size();
    if (nranks <= 1) return L;
    if (L < 2) throw SetupError{-1, "a single-level hierarchy cannot be distributed (problem too small)"};
    int lg = 1;
    while (lg < L - 1 && H.levels[lg].A.nrows >= gather_below) ++lg;
    return std::min(lg, L - 1);
}

std::vector<std::vector<int64_t>> level_starts(const HostHierarchy& H, int nranks, int lg) {
    const int L = (int)H.levels.size();
    const int top = std::min(lg, L - 1);
    std::vector<std::vector<int64_t>> st(top + 1, std::vector<int64_t>(nranks + 1, 0));
    const int64_t n0 = H.levels[0].A.nrows;
    for (int r = 0; r <= nranks; ++r) st[0][r] = (n0 * r) / nranks;
    for (int l = 0; l < top; ++l) {
        const auto& root = H.levels[l].root;
        if (!std::is_sorted(root.begin(), root.end()))
            throw SetupError{-1, "aggregate roots not ascending: cannot partition level " + std::to_string(l + 1)};
        for (int r = 0; r <= nranks; ++r)
            st[l + 1][r] = std::lower_bound(root.begin(), root.end(), st[l][r]) - root.begin();
    }
    return st;
}

namespace {

// outside columns of rows [r0, r1) of M that fall outside [lo, hi)
void outside_cols(const Csr& M, int64_t r0, int64_t r1, int64_t lo, int64_t hi, std::vector<int64_t>& out) {
    for (int64_t i = r0; i < r1; ++i)
        for (int64_t k = M.ptr[i]; k < M.ptr[i + 1]; ++k) {
            const int64_t c = M.col[k];
            if (c < lo || c >= hi) out.push_back(c);
        }
}

std::vector<int64_t> ghosts_of(const HostHierarchy& H, const std::vector<std::vector<int64_t>>& st, int l, int q) {
    const int L = (int)H.levels.size();
    const int64_t lo = st[l][q], hi = st[l][q + 1];
    std::vector<int64_t> g;
    outside_cols(H.levels[l].A, lo, hi, lo, hi, g);
    if (l < L - 1) outside_cols(H.levels[l].R, st[l + 1][q], st[l + 1][q + 1], lo, hi, g);
    if (l >= 1) outside_cols(H.levels[l - 1].P, st[l - 1][q], st[l - 1][q + 1], lo, hi, g);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    return g;
}

struct Numbering {  // global -> local of one distributed level
    int64_t lo = 0, hi = 0;
    const std::vector<int64_t>* ghosts = nullptr;
    bool identity = false;  // replicated level: global numbering
    int32_t operator()(int64_t c) const {
        if (identity) return (int32_t)c;
        if (c >= lo && c < hi) return (int32_t)(c - lo);
        auto it = std::lower_bound(ghosts->begin(), ghosts->end(), c);
        if (it == ghosts->end() || *it != c) throw std::logic_error("column missing from ghost list");
        return (int32_t)((hi - lo) + (it - ghosts->begin()));
    }
};

Csr extract_rows(const Csr& M, int64_t r0, int64_t r1, const Numbering& num, int64_t ncols_local) {
    Csr out;
    out.nrows = r1 - r0;
    out.ncols = ncols_local;
    out.ptr.assign(out.nrows + 1, 0);
    for (int64_t i = r0; i < r1; ++i) out.ptr[i - r0 + 1] = out.ptr[i - r0] + (M.ptr[i + 1] - M.ptr[i]);
    out.col.resize(out.ptr.back());
    out.val.resize(out.ptr.back());
    for (int64_t i = r0; i < r1; ++i) {
        int64_t d = out.ptr[i - r0];
        for (int64_t k = M.ptr[i]; k < M.ptr[i + 1]; ++k, ++d) {
            out.col[d] = num(M.col[k]);  // global entry order kept
            out.val[d] = M.val[k];
        }
    }
    return out;
}

}  // namespace

RankPart build_rank_part(const HostHierarchy& H, int nranks, int rank, int lg,
                         const std::vector<std::vector<int64_t>>& st) {
    const int L = (int)H.levels.size();
    RankPart RP;
    RP.rank = rank;
    RP.nranks = nranks;
    RP.lg = lg;
    RP.lv.resize(L);
    std::vector<std::vector<int64_t>> G(L);
    std::vector<Numbering> num(L);
    for (int l = 0; l < L; ++l) {
        if (l < lg && nranks > 1) {
            G[l] = ghosts_of(H, st, l, rank);
            num[l].lo = st[l][rank];
            num[l].hi = st[l][rank + 1];
            num[l].ghosts = &G[l];
        } else {
            num[l].identity = true;
        }
    }
    for (int l = 0; l < L; ++l) {
        const HostLevel& hl = H.levels[l];
        LevelPart& lp = RP.lv[l];
        const bool coarsest = l == L - 1;
        if (l >= lg || nranks == 1) {  // replicated (one rank: the whole level, no renumbering)
            lp.replicated = true;
            lp.row0 = 0;
            lp.row1 = hl.A.nrows;
            if (nranks == 1)
                lp.pA = &hl.A;
            else
                lp.A = hl.A;
            if (!coarsest) {
                if (nranks == 1) {
                    lp.pP = &hl.P;
                    lp.pR = &hl.R;
                } else {
                    lp.P = hl.P;
                    lp.R = hl.R;
                }
                lp.crow0 = 0;
                lp.crow1 = hl.P.ncols;
                lp.next_replicated = true;
            }
            lp.m = hl.m;
            lp.diag = hl.diag;
            lp.halo.nloc = hl.A.nrows;
            continue;
        }
        const int64_t lo = st[l][rank], hi = st[l][rank + 1], nloc = hi - lo;
        const int64_t ng = (int64_t)G[l].size();
        lp.row0 = lo;
        lp.row1 = hi;
        lp.A = extract_rows(hl.A, lo, hi, num[l], nloc + ng);
        if (!coarsest) {
            lp.crow0 = st[l + 1][rank];
            lp.crow1 = st[l + 1][rank + 1];
            lp.next_replicated = (l + 1 >= lg);
            const int64_t nc_cols = lp.next_replicated ? H.levels[l + 1].A.nrows
                                                       : (lp.crow1 - lp.crow0) + (int64_t)G[l + 1].size();
            lp.P = extract_rows(hl.P, lo, hi, num[l + 1], nc_cols);
            lp.R = extract_rows(hl.R, lp.crow0, lp.crow1, num[l], nloc + ng);
            auto take = [&](const std::vector<double>& v, std::vector<double>& out) {
                if (v.empty()) return;
                out.resize(nloc + ng);
                for (int64_t i = 0; i < nloc; ++i) out[i] = v[lo + i];
                for (int64_t g = 0; g < ng; ++g) out[nloc + g] = v[G[l][g]];
            };
            take(hl.m, lp.m);
            take(hl.diag, lp.diag);
        }
        // halo plan
        HaloPlan& hp = lp.halo;
        hp.nloc = nloc;
        hp.nghost = ng;
        hp.ghost_global = G[l];
        for (int64_t g = 0; g < ng;) {
            const int64_t c = G[l][g];
            const int owner = (int)(std::upper_bound(st[l].begin(), st[l].end(), c) - st[l].begin()) - 1;
            int64_t e = g;
            while (e < ng && G[l][e] < st[l][owner + 1]) ++e;
            hp.recv_peer.push_back(owner);
            hp.recv_off.push_back(g);
            hp.recv_cnt.push_back(e - g);
            g = e;
        }
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            const std::vector<int64_t> gq = ghosts_of(H, st, l, q);
            const int64_t off = (int64_t)hp.send_idx.size();
            for (int64_t c : gq)
                if (c >= lo && c < hi) hp.send_idx.push_back((int32_t)(c - lo));
            const int64_t cnt = (int64_t)hp.send_idx.size() - off;
            if (cnt > 0) {
                hp.send_peer.push_back(q);
                hp.send_off.push_back(off);
                hp.send_cnt.push_back(cnt);
            }
        }
    }
    return RP;
}

std::vector<LevelMeta> level_meta(const HostHierarchy& H) {
    std::vector<LevelMeta> m(H.levels.size());
    for (size_t l = 0; l < H.levels.size(); ++l) {
        const HostLevel& hl = H.levels[l];
        const bool coarsest = l + 1 == H.levels.size();
        m[l].rows = hl.A.nrows;
        m[l].nnz_A = hl.A.nnz();
        m[l].nnz_P = coarsest ? 0 : hl.P.nnz();
        m[l].cols_P = coarsest ? 0 : hl.P.ncols;
        m[l].n_agg = coarsest ? 0 : hl.n_agg;
        m[l].lmax = hl.lmax;
        m[l].lmin = hl.lmin;
        m[l].cheb_d = hl.cheb_d;
        m[l].cheb_c = hl.cheb_c;
    }
    return m;
}

namespace {

struct Writer {
    std::vector<uint8_t>& b;
    template <class T>
    void put(const T& v) {
        const auto* p = reinterpret_cast<const uint8_t*>(&v);
        b.insert(b.end(), p, p + sizeof(T));
    }
    template <class V>
    void vec(const V& v) {
        put<int64_t>((int64_t)v.size());
        const auto* p = reinterpret_cast<const uint8_t*>(v.data());
        b.insert(b.end(), p, p + v.size() * sizeof(typename V::value_type));
    }
    void csr(const Csr& M) {
        put(M.nrows);
        put(M.ncols);
        vec(M.ptr);
        vec(M.col);
        vec(M.val);
    }
};

struct Reader {
    const uint8_t* p;
    const uint8_t* end;
    void need(size_t n) const {
        if ((size_t)(end - p) < n) throw SetupError{-1, "scattered setup: truncated part image"};
    }
    template <class T>
    T get() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
    template <class V>
    void vec(V& v) {
        const int64_t n = get<int64_t>();
        if (n < 0) throw SetupError{-1, "scattered setup: bad part image"};
        const size_t bytes = (size_t)n * sizeof(typename V::value_type);
        need(bytes);
        v.resize(n);
        if (bytes) std::memcpy(v.data(), p, bytes);
        p += bytes;
    }
    void csr(Csr& M) {
        M.nrows = get<int64_t>();
        M.ncols = get<int64_t>();
        vec(M.ptr);
        vec(M.col);
        vec(M.val);
    }
};

constexpr uint64_t kPartMagic = 0x414d4742504152ULL;  // "AMGBPAR"

}  // namespace

void pack_part(const PartHeader& hd, const RankPart& rp, std::vector<uint8_t>& out) {
    out.clear();
    Writer w{out};
    w.put(kPartMagic);
    w.vec(hd.meta);
    w.put<int32_t>(hd.lg);
    w.put<int64_t>((int64_t)hd.starts.size());
    for (const auto& st : hd.starts) w.vec(st);
    w.vec(hd.coarse_inv);
    w.put<int32_t>(rp.rank);
    w.put<int32_t>(rp.nranks);
    w.put<int32_t>(rp.lg);
    w.put<int64_t>((int64_t)rp.lv.size());
    for (const LevelPart& lp : rp.lv) {
        w.put<int32_t>(lp.replicated);
        w.put<int32_t>(lp.next_replicated);
        w.put(lp.row0);
        w.put(lp.row1);
        w.put(lp.crow0);
        w.put(lp.crow1);
        w.csr(lp.ma());
        w.csr(lp.mp());
        w.csr(lp.mr());
        const HaloPlan& h = lp.halo;
        w.put(h.nloc);
        w.put(h.nghost);
        w.vec(h.ghost_global);
        w.vec(h.recv_peer);
        w.vec(h.recv_off);
        w.vec(h.recv_cnt);
        w.vec(h.send_peer);
        w.vec(h.send_off);
        w.vec(h.send_cnt);
        w.vec(h.send_idx);
        w.vec(lp.m);
        w.vec(lp.diag);
    }
    w.put(kPartMagic);
}

void unpack_part(const uint8_t* p, size_t n, PartHeader& hd, RankPart& rp) {
    Reader r{p, p + n};
    if (r.get<uint64_t>() != kPartMagic) throw SetupError{-1, "scattered setup: bad part image"};
    r.vec(hd.meta);
    hd.lg = r.get<int32_t>();
    hd.starts.resize(r.get<int64_t>());
    for (auto& st : hd.starts) r.vec(st);
    r.vec(hd.coarse_inv);
    rp.rank = r.get<int32_t>();
    rp.nranks = r.get<int32_t>();
    rp.lg = r.get<int32_t>();
    rp.lv.resize(r.get<int64_t>());
    for (LevelPart& lp : rp.lv) {
        lp.replicated = r.get<int32_t>() != 0;
        lp.next_replicated = r.get<int32_t>() != 0;
        lp.row0 = r.get<int64_t>();
        lp.row1 = r.get<int64_t>();
        lp.crow0 = r.get<int64_t>();
        lp.crow1 = r.get<int64_t>();
        r.csr(lp.A);
        r.csr(lp.P);
        r.csr(lp.R);
        HaloPlan& h = lp.halo;
        h.nloc = r.get<int64_t>();
        h.nghost = r.get<int64_t>();
        r.vec(h.ghost_global);
        r.vec(h.recv_peer);
        r.vec(h.recv_off);
        r.vec(h.recv_cnt);
        r.vec(h.send_peer);
        r.vec(h.send_off);
        r.vec(h.send_cnt);
        r.vec(h.send_idx);
        r.vec(lp.m);
        r.vec(lp.diag);
    }
    if (r.get<uint64_t>() != kPartMagic || r.p != r.end) throw SetupError{-1, "scattered setup: bad part image"};
}

}  // namespace amgb

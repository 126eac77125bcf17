// Upload of one level's host index data (host/topology.hpp) into a device Level.
#include <algorithm>
#include <atomic>

#include "level.cuh"

namespace ksb {

void upload_level(Ctx& cx, std::shared_ptr<FineTopology> topo, Level& L) {
    static std::atomic<uint64_t> next_uid{1};
    L.ctx = &cx;
    L.uid = next_uid.fetch_add(1);
    L.topo = std::move(topo);
    const auto& T = *L.topo;
    const auto& S = *T.space;
    const auto& M = *S.mesh;
    L.n = S.n();
    L.ni = S.ni();
    L.nb = S.nb();
    L.nt = M.n_tets();
    L.nnz_ii = T.ii.nnz();
    L.nnz_ib = T.ib.nnz();
    L.nH = T.coarse->ni();
    L.nct = T.coarse->mesh->n_tets();
    L.ncv = T.coarse->n();
    L.xyz.upload(cx, M.xyz);
    L.tets.upload(cx, M.tets);
    L.interior.upload(cx, S.interior);
    L.boundary.upload(cx, S.boundary);
    L.iidx.upload(cx, S.iidx);
    L.ii_ptr.upload(cx, T.ii.ptr);
    L.ii_col.upload(cx, T.ii.col);
    L.ib_ptr.upload(cx, T.ib.ptr);
    L.ib_col.upload(cx, T.ib.col);
    L.diag_slot.upload(cx, T.diag_slot);
    L.ii_gptr.upload(cx, T.ii_gptr);
    L.ii_gent.upload(cx, T.ii_gent);
    L.ib_gptr.upload(cx, T.ib_gptr);
    L.ib_gent.upload(cx, T.ib_gent);
    L.pint_col.upload(cx, T.pint_col);
    L.pint_val.upload(cx, T.pint_val);
    L.ancestor.upload(cx, T.ancestor);
    L.anc_ptr.upload(cx, T.anc_ptr);
    L.anc_tets.upload(cx, T.anc_tets);
    {
        // K-PROJ chunks: at most `cap` fine tets each, so that a coarse tet holding most of an adaptive level's
        // tets (near a nucleus) is spread over many blocks; uniform levels (nt / nct <= cap) keep one per coarse tet
        const int nct = std::max(0, int(T.anc_ptr.size()) - 1);
        const int64_t cap = std::max<int64_t>(1024, (int64_t(T.anc_tets.size()) + 2047) / 2048);
        std::vector<int32_t> cc, cb, ce, cp(size_t(nct) + 1, 0);
        for (int C = 0; C < nct; ++C) {
            cp[size_t(C)] = int32_t(cc.size());
            const int32_t b = T.anc_ptr[size_t(C)], e = T.anc_ptr[size_t(C) + 1];
            const int64_t pieces = std::max<int64_t>(1, (int64_t(e - b) + cap - 1) / cap);
            for (int64_t q = 0; q < pieces; ++q) {
                cc.push_back(C);
                cb.push_back(int32_t(b + (int64_t(e - b) * q) / pieces));
                ce.push_back(int32_t(b + (int64_t(e - b) * (q + 1)) / pieces));
            }
        }
        if (!T.anc_ptr.empty()) cp[size_t(nct)] = int32_t(cc.size());
        L.pj_n = int(cc.size());
        L.pj_c.upload(cx, cc);
        L.pj_b.upload(cx, cb);
        L.pj_e.upload(cx, ce);
        L.pj_ptr.upload(cx, cp);
    }
    L.vinc_ptr.upload(cx, T.vinc_ptr);
    L.vinc.upload(cx, T.vinc);
    L.bvinc_ptr.upload(cx, T.bvinc_ptr);
    L.bvinc.upload(cx, T.bvinc);
    L.cinc_ptr.upload(cx, T.cinc_ptr);
    L.cinc.upload(cx, T.cinc);
    L.ctets.upload(cx, T.coarse->mesh->tets);
    L.ciidx.upload(cx, T.coarse->iidx);
    L.cxyz.upload(cx, T.coarse->mesh->xyz);
    L.sell_ptr.upload(cx, T.sell_ptr);
    L.sell_col.upload(cx, T.sell_col);
    L.sell_map.upload(cx, T.sell_map);
    L.t8_col.upload(cx, T.t8_col);
    L.t8_map.upload(cx, T.t8_map);
    L.lo_perm.upload(cx, T.lo_perm);
    L.lo_ptr.upload(cx, T.lo_ptr);
    L.lo_col.upload(cx, T.lo_col);
    L.lo_map.upload(cx, T.lo_map);
    L.lo_dslot.upload(cx, T.lo_dslot);
    L.lo_max_row = T.lo_max_row;
    L.ut_rows.upload(cx, T.ut_rows);
    L.ut_eptr.upload(cx, T.ut_eptr);
    L.ut_ent.upload(cx, T.ut_ent);
    L.ut_map.upload(cx, T.ut_map);
    L.ut_nt = T.ut_nt;
    L.dia_ng = T.dia_ng;
    L.dia_lr = T.dia_lr;
    L.dia_lo = T.dia_lo;
    L.dia_n = T.dia_n;
    for (int q = 0; q < T.dia_ng; ++q) L.dia_first[q] = T.dia_first[q];
    L.nslices = int(T.sell_ptr.size()) - 1;
    L.max_row_ii = 0;
    for (size_t i = 0; i + 1 < T.ii.ptr.size(); ++i) L.max_row_ii = std::max(L.max_row_ii, int(T.ii.ptr[i + 1] - T.ii.ptr[i]));
    L.n_prev = T.n_prev;
    if (T.n_prev > 0) {
        L.pstep_col.upload(cx, T.pstep_col);
        L.pstep_val.upload(cx, T.pstep_val);
        L.prev_iidx.upload(cx, T.prev_iidx);
    }
    for (int d = 0; d < 3; ++d) {
        L.box_lo[d] = M.lo[d];
        L.box_hi[d] = M.hi[d];
    }
}

} // namespace ksb

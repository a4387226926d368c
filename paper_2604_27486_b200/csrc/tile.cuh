/* tile.cuh -- the data-parallel form of the post-SSA stage: one CTA keeps a
 * *tile* (a run of consecutive small functions, ~1000 records) resident in
 * shared memory and takes all of them through the passes together, one
 * thread per instruction record / candidate / selected match:
 *
 *   use counts + def positions (smem atomics)
 *   seed classes (per-block class counts)  -> FindSeeds  patterns.py:189-191
 *   join unification per (pattern, anchor) -> Unify      patterns.py:130-216
 *   overlap selection (atomicMin bidding)  -> select_matches :241-252
 *   rewrite planning, id allocation by segmented scans, in-place
 *   permutation of the stream              -> _apply_patterns :671-707
 *   pack simplification, dead-pseudo fixpoint, reciprocal chains, tagging
 *
 * HBM sees one coalesced read of the tile and one write of the result; every
 * intermediate round lives in shared memory.
 *
 * Ids: value, immediate and memref indices are function-local in the corpus.
 * On load they are rebased into tile-wide index spaces (each function gets a
 * slice with room to grow), so ONE function state (`FS`, in shared memory)
 * describes the whole tile and the per-match leaf code of core.cuh (the nine
 * rewrite planners) runs on it unchanged; the store rebases them back.
 *
 * Exactness: the reference is sequential over blocks and chains.  Everything
 * here is evaluated on the snapshot taken at the start of a pass, which equals
 * the sequential result unless a later item observes an earlier item's edit.
 * Those cases (G5 cross-block escapes, interfering reciprocal chains, RZ/PT
 * join links, capacity, reference exceptions) are *detected* and the function
 * is handed, untouched, to the general per-function kernel of core.cuh.
 */
#pragma once
#include "core.cuh"
#include "kargs.h"
#if !CL_DEV
#include <stdio.h>
#include <stdlib.h>
#endif

namespace clk {

/* the two unify helpers: out of line by default (code size; the stage was instruction-fetch bound in round 1) */
#ifdef CL_INLINE_UNIFY
#define CLU CLD
#else
#define CLU CLN
#endif

/* a record removed by remove_dead_pseudo stays in place as a tombstone (no arities, no guard, an opcode id no table
 * ever hands out: layout.py caps ids below 0xFFFF) until the next rewrite permutation or the store drops it: no
 * compaction pass, positions and def-use stay valid                                                            */
static constexpr uint16_t CL_OP_TOMB = 0xFFFF;
static constexpr uint32_t CL_ST_REDO = 100;     /* internal: redo this function on the general kernel */


struct TMatch { uint16_t pos[3]; uint8_t pat, n; };
struct TChain { uint16_t add, mufu; uint32_t rcp, addv; uint8_t f, ok; uint16_t rank; };
/* unification of one pattern as equality constraints between operand slots:
 * every later occurrence of a variable must carry the key of its first one
 * (Bindings.bind, patterns.py:93-97), same for the "mod:<var>" bindings (:163-166) */
struct TPat {
    uint8_t n_pairs, n_mpairs, pad[2];
    uint8_t pair[28][4];       /* tA, kA, tB, kB: slots in defs, aux, uses order    */
    uint8_t mpair[4][4];       /* tA, groupA, tB, groupB                            */
};

/* capacities of one tile (compile time: the tile lives in shared memory) */
struct TileCfgL { static constexpr bool PP = false; static constexpr uint32_t I = 1024, V = 1792, Q = 320, F = 32, B = 96, M = 1024, S = 512, X = 256, E = 512; };
/* a big tile resident in L2 (global scratch) instead of shared memory: every pass loops many times over
 * the same code, which is what the instruction cache needs (profiles/r01_tuning.md)          */
struct TileCfgG { static constexpr bool PP = true; static constexpr uint32_t I = 4096, V = 7168, Q = 1280, F = 128, B = 255, M = 4096, S = 2048, X = 512, E = 2048; };
struct TileCfgG2 { static constexpr bool PP = true; static constexpr uint32_t I = 8192, V = 14336, Q = 2560, F = 255, B = 255, M = 8192, S = 4096, X = 1024, E = 4096; };
struct TileCfgG3 { static constexpr bool PP = true; static constexpr uint32_t I = 16384, V = 28672, Q = 5120, F = 255, B = 255, M = 16384, S = 8192, X = 2048, E = 8192; };

/* one long unrolled block per tile: a 16 384-instruction block is ~19 500 records (positions stay below 65 536) */
struct TileCfgG4 { static constexpr bool PP = true; static constexpr uint32_t I = 32768, V = 57344, Q = 10240, F = 255, B = 255, M = 32768, S = 16384, X = 4096, E = 16384; };

/* the pattern table and what t_setup derives from it: shared by the tiles of a CTA */
struct TileP {
    cl_pattern_blob pb;
    TPat pat[CL_MAX_PATTERNS];
    uint16_t cls_op[2][MAX_CLS];
    uint32_t n_cls[2], anchor_mask[2][MAX_CLS];
    uint8_t op_cls[2][CL_OP__COUNT];      /* opcode id -> seed class of the table, 0xFF none */
};

/* a plane of the tile's stream: an array inside the tile (shared-memory tiles, permuted through registers) or a
 * pair of buffers in scratch that a permutation flips (big tiles: the stream is written once per permutation
 * instead of being scattered to a side buffer and copied back -- half the DRAM traffic of a permutation)      */
template <class E, uint32_t N, bool PP> struct PlaneT;
template <class E, uint32_t N> struct PlaneT<E, N, false> {
    alignas(16) E a[N];
    CLMEM E &operator[](size_t i) { return a[i]; }
    CLMEM const E &operator[](size_t i) const { return a[i]; }
    CLMEM E *ptr() { return a; }
};
template <class E, uint32_t N> struct PlaneT<E, N, true> {
    E *a, *b;
    CLMEM E &operator[](size_t i) { return a[i]; }
    CLMEM const E &operator[](size_t i) const { return a[i]; }
    CLMEM E *ptr() { return a; }
    CLMEM void flip() { E *t = a; a = b; b = t; }
};
template <class C> struct TileS {
    PlaneT<cl_hdr, C::I, C::PP> hdr;
    PlaneT<uint16_t, C::I * 8, C::PP> tag;
    PlaneT<uint32_t, C::I * 8, C::PP> pay;
    unsigned long long owner[C::I];
    uint32_t usecnt[C::V], defpos[C::V], redirect[C::V], origin[C::V];
    int32_t def_iid[C::V];
    cl_imm imm[C::Q];
    SelRec sel[C::S];
    TMatch mt[C::M];
    TChain chain[C::X];
    uint16_t outpos[C::I], sel_at[C::I];
    uint8_t keep[C::I], inscnt[C::I], clsid[C::I], flag[C::I];
    /* function / block index of every record: moved along by the permutations of a big tile (a second buffer
     * each), recomputed from the block offsets (t_index) in a shared-memory tile                             */
    PlaneT<uint8_t, C::I, C::PP> fidx, bidx;
    uint8_t alive[C::V];
    uint8_t mstate[C::M];
    /* blocks */
    uint32_t bo[C::B + 1], bo2[C::B + 1], b_first[C::B];
    cl_blk blk[C::B];
    uint32_t ccnt[C::B][MAX_CLS];
    uint32_t cbase[C::B][MAX_CLS];          /* over-budget blocks: members of the class before the block (tile wide count) */
    uint16_t b_over[C::B];                  /* classes of the block whose product order must be computed exactly */
    uint8_t bfun[C::B];
    /* functions: slices of the tile-wide value / immediate / memref index spaces */
    uint32_t f_vbase[C::F + 1], f_qbase[C::F + 1], f_mbase[C::F + 1];
    uint32_t f_nvid[C::F], f_niid[C::F], f_nimm[C::F], f_ntemp[C::F], f_stat[C::F], f_nev[C::F];
    uint32_t f_b0[C::F + 1], f_i0[C::F + 1], f_gf[C::F], f_gb0[C::F], f_gi0[C::F];   /* tile block / record ranges; global function, block, record */
    uint32_t f_chg[C::F], f_red[C::F], f_first[C::F], f_aux[C::F], f_nin[C::F];
    uint32_t f_oi[C::F], f_oq[C::F], f_ov[C::F], f_oe[C::F];
    uint32_t f_stats[C::F][64];
    uint8_t f_arch[C::F], f_active[C::F], f_odd[C::F], f_gate[C::F], f_rgate[C::F];
    /* the one function state of the tile + tile scalars */
    const struct TileP *P;
    FS fs;
    unsigned long long prof[PF__N];
    uint32_t n, nb, nf, n_mt, n_sel, n_ev, fail, vtot, qtot, n_chain, work;
    uint32_t du_ok, n_list;       /* du_ok: usecnt / defpos describe the stream (every live function) */
    uint32_t tombs;               /* the stream holds tombstones */
    uint32_t red[40];
    uint32_t pcnt[CL_MAX_PATTERNS], pcur[CL_MAX_PATTERNS];     /* t_sort_by_pattern: items per pattern, fill cursors */
};

template <class C> struct TileG {      /* what lives outside shared memory */
    Stage *stage;             /* [C::S] staged rewrites (L2-resident scratch)   */
    cl_event *ev;             /* [C::E]                                          */
    cl_memref *mem;           /* memrefs of the tile: mutable copy in the output  */
    Rec *tmp;                 /* [C::I] second stream buffer of tiles too big to permute in registers, else null */
};

template <class C> CLD bool tf_ok(const TileS<C> &T, uint32_t f) { return *(volatile const uint32_t *)&T.f_stat[f] == 0; }
template <class C> CLD void tf_fail(TileS<C> &T, uint32_t f, uint32_t code) { a_cas0(&T.f_stat[f], code); }

template <class C> CLD void t_event(TileS<C> &T, const TileG<C> &tg, uint32_t f, uint32_t seq, uint32_t kind,
                                    uint32_t idx, uint32_t a, uint32_t b) {
    const uint32_t k = a_add(&T.n_ev, 1u);
    if (k < C::E) {
        cl_event e; e.func = f;      /* tile-local: t_store writes the global id */ e.seq = seq; e.kind = kind; e.idx = idx; e.a = a; e.b = b; e.c = 0; e.d = 0;
        tg.ev[k] = e;
        a_add(&T.f_nev[f], 1u);
    } else
        T.fail = 1;
}

template <class C> CLD int t_class_of(const TileS<C> &T, unsigned table, uint16_t op) {
    if (op >= CL_OP__COUNT) return -1;            /* dynamic opcodes never head a template */
    const uint8_t c = T.P->op_cls[table][op];
    return c == 0xFF ? -1 : (int)c;
}
/* operand slot k (guard included) of a record without overflow slots           */
template <class C> CLD opnd t_slot(const TileS<C> &T, uint32_t i, unsigned k) {
    opnd o; o.tag = T.tag[(size_t)i * 8 + k]; o.pay = T.pay[(size_t)i * 8 + k];
    return o;
}
/* value_operands (ssa.py:599-610) / all_defs of a record without overflow slots */
template <class C, class F> CLD void t_value_operands(const TileS<C> &T, const TileG<C> &tg, const cl_hdr &h, uint32_t i, F fn) {
    if (has_guard(h)) { const opnd g = t_slot(T, i, 0); if (is_value(g)) fn(g.pay); }
    const unsigned u0 = use0(h);
    for (unsigned k = 0; k < h.n_uses; k++) {
        const opnd u = t_slot(T, i, u0 + k);
        if (is_value(u)) fn(u.pay);
        else if (kind_of(u.tag) == CL_K_MEMREF) {
            const cl_memref &m = tg.mem[u.pay];
            if (kind_of(m.base_tag) == CL_K_VALUE) fn(m.base_pay);
            if (kind_of(m.ureg_tag) == CL_K_VALUE) fn(m.ureg_pay);
        }
    }
}
template <class C, class F> CLD void t_value_defs(const TileS<C> &T, const cl_hdr &h, uint32_t i, F fn) {
    const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
    for (unsigned k = 0; k < nd; k++) { const opnd d = t_slot(T, i, d0 + k); if (is_value(d)) fn(d.pay); }
}

/* block / function index of every record from the block offsets */
template <class G, class C> CLF void t_index(const G &g, TileS<C> &T) {
    GFOR(g, i, T.n) if (i < T.n) {
        uint32_t lo = 0, hi = T.nb;                  /* last b with bo[b] <= i */
        while (lo + 1 < hi) { const uint32_t mid = (lo + hi) >> 1; if (T.bo[mid] <= i) lo = mid; else hi = mid; }
        T.bidx[i] = (uint8_t)lo; T.fidx[i] = T.bfun[lo];
    }
    g.sync();
}

/* def-use contribution of one record that now sits at position `at` (ssa.build_defuse, ssa.py:613-636): what
 * t_usecount does per record, from the record's four 128-bit words while a permutation has them in registers
 * (slots addressed with compile-time indices: no local memory).  Records of tiles have no overflow slots.     */
template <class C> CLD void t_du_record(TileS<C> &T, const TileG<C> &tg, const uint4 &r0, const uint4 &r1, const uint4 &r2, const uint4 &r3,
                                        uint32_t at, uint32_t f) {
    const uint32_t w2 = r0.z;                                   /* n_defs, n_aux, n_uses, flags (cl_hdr bytes 8..11) */
    const unsigned nd = w2 & 0xFFu, na = (w2 >> 8) & 0xFFu, nu = (w2 >> 16) & 0xFFu;
    const unsigned g0 = ((w2 >> 24) & CL_IF_GUARD) ? 1u : 0u, d_end = g0 + nd + na, u_end = d_end + nu;
    const uint32_t tw[4] = { r1.x, r1.y, r1.z, r1.w };
    const uint32_t pw[8] = { r2.x, r2.y, r2.z, r2.w, r3.x, r3.y, r3.z, r3.w };
    bool odd = false;
#pragma unroll
    for (unsigned k = 0; k < 8; k++) {
        if (k >= u_end) continue;
        const uint16_t tag = (uint16_t)(k & 1u ? tw[k >> 1] >> 16 : tw[k >> 1] & 0xFFFFu);
        const uint32_t pay = pw[k];
        const unsigned kd = kind_of(tag);
        if (k >= g0 && k < d_end) {                             /* defs and aux defs */
            if (kd == CL_K_VALUE) { if (pay < C::V) T.defpos[pay] = at; }
            else odd |= !(kd == CL_K_RZ || kd == CL_K_URZ || kd == CL_K_PRED);
        } else if (kd == CL_K_VALUE) {                          /* guard, uses */
            if (pay < C::V) a_add(&T.usecnt[pay], 1u);
        } else if (kd == CL_K_MEMREF && k >= d_end) {
            const cl_memref &m = tg.mem[pay];
            if (kind_of(m.base_tag) == CL_K_VALUE && m.base_pay < C::V) a_add(&T.usecnt[m.base_pay], 1u);
            if (kind_of(m.ureg_tag) == CL_K_VALUE && m.ureg_pay < C::V) a_add(&T.usecnt[m.ureg_pay], 1u);
        }
    }
    if (odd) T.f_odd[f] = 1;
}

/* in-place permutation of the stream: record i moves to dst(i) (NONE32 = dropped).
 * Everything is read before anything is written.  COUNT (big tiles): def positions and use counts of the moved
 * records are taken on the way (the caller has zeroed them and adds what it inserts): no recount sweep after.  */
template <bool COUNT = false, class G, class C, class F> CLD void t_permute(const G &g, TileS<C> &T, const TileG<C> &tg, uint32_t n, uint32_t n_new, F dst) {
    if constexpr (C::PP) {
        /* into the other buffer of every plane, then the buffers flip */
        GFOR(g, i, n) if (i < n) {
            const uint32_t d = dst(i);
            if (d != NONE32) {
                const uint4 r0 = *(const uint4 *)&T.hdr[i], r1 = *(const uint4 *)&T.tag[(size_t)i * 8];
                const uint4 r2 = ((const uint4 *)&T.pay[(size_t)i * 8])[0], r3 = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
                *(uint4 *)&T.hdr.b[d] = r0;
                *(uint4 *)&T.tag.b[(size_t)d * 8] = r1;
                ((uint4 *)&T.pay.b[(size_t)d * 8])[0] = r2;
                ((uint4 *)&T.pay.b[(size_t)d * 8])[1] = r3;
                const uint32_t f = T.fidx[i];
                T.fidx.b[d] = (uint8_t)f; T.bidx.b[d] = T.bidx[i];
                if (COUNT && tf_ok(T, f)) t_du_record(T, tg, r0, r1, r2, r3, d, f);
            }
        }
        g.sync();
        if (g.rank == 0) {
            T.hdr.flip(); T.tag.flip(); T.pay.flip(); T.fidx.flip(); T.bidx.flip();
            T.fs.S.hdr = T.hdr.ptr(); T.fs.S.tag = T.tag.ptr(); T.fs.S.pay = T.pay.ptr();
        }
        g.sync();
        (void)tg; (void)n_new;
        return;
    } else {
#if CL_DEV
    constexpr int K = (int)((C::I + G::THREADS - 1) / G::THREADS);
    if (K > 2) {
        /* through the second buffer: scatter, then copy back */
        GFOR(g, i, n) if (i < n) {
            const uint32_t d = dst(i);
            if (d != NONE32) {
                uint4 *o = (uint4 *)&tg.tmp[d];
                o[0] = *(const uint4 *)&T.hdr[i];
                o[1] = *(const uint4 *)&T.tag[(size_t)i * 8];
                o[2] = ((const uint4 *)&T.pay[(size_t)i * 8])[0];
                o[3] = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
            }
        }
        g.sync();
        GFOR(g, i, n_new) if (i < n_new) {
            const uint4 *r = (const uint4 *)&tg.tmp[i];
            *(uint4 *)&T.hdr[i] = r[0];
            *(uint4 *)&T.tag[(size_t)i * 8] = r[1];
            ((uint4 *)&T.pay[(size_t)i * 8])[0] = r[2];
            ((uint4 *)&T.pay[(size_t)i * 8])[1] = r[3];
        }
        g.sync();
        return;
    }
    constexpr int KR = K > 2 ? 1 : K;
    uint4 r[KR][4];
    uint32_t d[KR];
#pragma unroll
    for (int k = 0; k < KR; k++) {
        const uint32_t i = (uint32_t)k * g.size + g.rank;
        d[k] = i < n ? dst(i) : NONE32;
        if (d[k] != NONE32) {
            r[k][0] = *(const uint4 *)&T.hdr[i];
            r[k][1] = *(const uint4 *)&T.tag[(size_t)i * 8];
            r[k][2] = ((const uint4 *)&T.pay[(size_t)i * 8])[0];
            r[k][3] = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
        }
    }
    g.sync();
#pragma unroll
    for (int k = 0; k < KR; k++)
        if (d[k] != NONE32) {
            const uint32_t o = d[k];
            *(uint4 *)&T.hdr[o] = r[k][0];
            *(uint4 *)&T.tag[(size_t)o * 8] = r[k][1];
            ((uint4 *)&T.pay[(size_t)o * 8])[0] = r[k][2];
            ((uint4 *)&T.pay[(size_t)o * 8])[1] = r[k][3];
        }
    g.sync();
#else
    static Rec tmp[C::I];
    static uint32_t d[C::I];
    for (uint32_t i = 0; i < n; i++) {
        d[i] = dst(i);
        if (d[i] != NONE32) { tmp[i].h = T.hdr[i]; memcpy(tmp[i].tag, &T.tag[(size_t)i * 8], 16); memcpy(tmp[i].pay, &T.pay[(size_t)i * 8], 32); }
    }
    for (uint32_t i = 0; i < n; i++)
        if (d[i] != NONE32) { T.hdr[d[i]] = tmp[i].h; memcpy(&T.tag[(size_t)d[i] * 8], tmp[i].tag, 16); memcpy(&T.pay[(size_t)d[i] * 8], tmp[i].pay, 32); }
    (void)g; (void)tg; (void)n_new;
#endif
    }
}

/* running exclusive scan over items [0, n) in order; returns the total        */
template <class G, class FIN, class FOUT> CLD uint32_t t_scan(const G &g, uint32_t n, FIN in, FOUT out) {
    /* every lane owns a contiguous run of items: its sum, ONE scan of the sums over the group, then the run again.
     * (Round 1 scanned chunk by chunk, two barriers per 1024 items: a 12 000-record tile paid 24 per scan.)   */
    const uint32_t per = (n + g.size - 1) / g.size;
    const uint32_t lo = g.rank * per < n ? g.rank * per : n, hi = lo + per < n ? lo + per : n;
    uint32_t sum = 0;
    for (uint32_t j = lo; j < hi; j++) sum += in(j);
    uint32_t total;
    uint32_t run = g.exscan(sum, total);
    for (uint32_t j = lo; j < hi; j++) { const uint32_t x = in(j); out(j, run); run += x; }
    return total;
}

/* new block offsets after a permutation described by outpos[] (position of the
 * first output slot of every old record) and the new length                   */
template <class G, class C> CLD void t_rebase_blocks(const G &g, TileS<C> &T, uint32_t n_old, uint32_t n_new) {
    GFOR(g, b, T.nb + 1) if (b <= T.nb) { const uint32_t old = T.bo[b]; T.bo2[b] = old < n_old ? (uint32_t)T.outpos[old] : n_new; }
    g.sync();
    GFOR(g, b, T.nb + 1) if (b <= T.nb) T.bo[b] = T.bo2[b];
    if (g.rank == 0) { T.n = n_new; T.du_ok = 0; }
    g.sync();
}

/* ------------------------------------------------------------------ def-use */
/* ssa.py:613-636 for every live function of the tile at once                  */
template <class G, class C> CLF void t_usecount(const G &g, TileS<C> &T, const TileG<C> &tg) {
    PROF(g, T.fs, PF_USECOUNT);
    GFOR(g, v, T.vtot) if (v < T.vtot) { T.usecnt[v] = 0; T.defpos[v] = NONE32; }
    g.sync();
    GFOR(g, i, T.n) if (i < T.n) {
        const uint32_t f = T.fidx[i];
        if (!tf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
        bool odd = false;
        for (unsigned k = 0; k < nd; k++) {
            const opnd d = t_slot(T, i, d0 + k);
            const unsigned kd = kind_of(d.tag);
            if (kd == CL_K_VALUE) { if (d.pay < C::V) T.defpos[d.pay] = i; }
            else odd |= !(kd == CL_K_RZ || kd == CL_K_URZ || kd == CL_K_PRED);
        }
        if (odd) T.f_odd[f] = 1;
        t_value_operands(T, tg, h, i, [&](uint32_t v) { if (v < C::V) a_add(&T.usecnt[v], 1u); });
    }
    GFOR(g, b, T.nb) if (b < T.nb) {
        if (!tf_ok(T, T.bfun[b])) continue;
        for (int k = 0; k < 2; k++)
            if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE && T.blk[b].term_pay[k] < C::V)
                a_add(&T.usecnt[T.blk[b].term_pay[k]], 1u);
    }
    if (g.rank == 0) T.du_ok = 1;
    g.sync();
}

/* ----------------------------------------------------------------- matching */
/* operand_key equality (patterns.py:109-127) of two operands                   */
template <class C> CLU bool t_key_equal(const TileS<C> &T, const TileG<C> &tg, opnd a, opnd b) {
    unsigned ka = kind_of(a.tag), kb = kind_of(b.tag);
    if (ka == CL_K_URZ) ka = CL_K_RZ;
    if (kb == CL_K_URZ) kb = CL_K_RZ;
    const bool oa = ka == CL_K_NONE || ka >= CL_K_MEMREF, ob = kb == CL_K_NONE || kb >= CL_K_MEMREF;
    if (oa || ob) {
        if (!(oa && ob)) return false;
        const cl_memref &x = tg.mem[a.pay], &y = tg.mem[b.pay];       /* ("other", str(op)) */
        if (x.base_tag != y.base_tag || x.ureg_tag != y.ureg_tag) return false;
        if (kind_of(x.base_tag) != CL_K_NONE && x.base_pay != y.base_pay) return false;
        if (kind_of(x.ureg_tag) != CL_K_NONE && x.ureg_pay != y.ureg_pay) return false;
        return x.off_hi == y.off_hi && x.off_lo == y.off_lo;
    }
    if (ka != kb) return false;
    if (ka == CL_K_RZ) return true;
    if (ka == CL_K_IMM) return T.imm[a.pay].bits == T.imm[b.pay].bits;
    return a.pay == b.pay;
}
/* _match_opcode + the slot-local part of _unify (patterns.py:155-178, :130-152) */
template <class C> CLU bool t_match_local(const TileS<C> &T, const cl_template &t, const cl_hdr &h, uint32_t i) {
    if (h.op != t.op) return false;
    const cl_modset &ms = T.fs.ms[h.modset];
    if ((ms.mask & t.mods_all) != t.mods_all) return false;
    if (ms.mask & t.mods_none) return false;
    for (unsigned k = 0; k < t.n_modvars; k++) if (ms.first[t.modvar_group[k]] == 0xFF) return false;
    if (t.n_defs != h.n_defs || t.n_aux != h.n_aux || t.n_uses != h.n_uses) return false;
    if (h.flags & CL_IF_EXT) return false;
    const unsigned n = (unsigned)t.n_defs + t.n_aux + t.n_uses, g0 = has_guard(h);
    for (unsigned k = 0; k < n; k++) {
        const cl_slot &sl = t.slot[k];
        if (sl.kind == CL_S_ANY) continue;
        const opnd o = t_slot(T, i, g0 + k);
        switch (sl.kind) {
        case CL_S_RZ: if (!is_zero(o)) return false; break;
        case CL_S_PT:
            if (!(kind_of(o.tag) == CL_K_PRED && o.pay == CL_PT_INDEX)) return false;
            if (sl.neg != 0 && o_neg(o) != (sl.neg == 2)) return false;
            break;
        case CL_S_IMM: if (!(is_imm(o) && T.imm[o.pay].bits == sl.imm)) return false; break;
        case CL_S_VAR:
            if (sl.neg && o_neg(o) != (sl.neg == 2)) return false;
            if (sl.bitnot && o_not(o) != (sl.bitnot == 2)) return false;
            if (sl.half && o_half(o) != sl.half) return false;
            break;
        default: return false;
        }
    }
    return true;
}
/* one candidate tuple of match_patterns (patterns.py:199-215)                  */
template <class C> CLD bool t_check_tuple(const TileS<C> &T, const TileG<C> &tg, unsigned pi, const uint32_t *idx) {
    const cl_pattern &p = T.P->pb.p[pi];
    const unsigned nt = p.n_templates;
    for (unsigned t = 0; t < nt; t++) if (!t_match_local(T, p.t[t], T.hdr[idx[t]], idx[t])) return false;
    const TPat &tp = T.P->pat[pi];
    for (unsigned q = 0; q < tp.n_mpairs; q++) {
        const uint8_t *m = tp.mpair[q];
        if (T.fs.ms[T.hdr[idx[m[0]]].modset].first[m[1]] != T.fs.ms[T.hdr[idx[m[2]]].modset].first[m[3]]) return false;
    }
    for (unsigned q = 0; q < tp.n_pairs; q++) {
        const uint8_t *m = tp.pair[q];
        const uint32_t ia = idx[m[0]], ib = idx[m[2]];
        if (!t_key_equal(T, tg, t_slot(T, ia, has_guard(T.hdr[ia]) + m[1]), t_slot(T, ib, has_guard(T.hdr[ib]) + m[3]))) return false;
    }
    /* _connected (patterns.py:219-238) holds by construction: every member but the anchor was found as the SSA
     * definition of a value operand of an already resolved member, so it shares that value with it (round 1
     * re-checked it here: 8.8 % of the kernel's instructions at 3.8 active lanes)                          */
    (void)tg;
    return true;
}

/* one (pattern, anchor) item of match_patterns (patterns.py:181-216), join form
 * (see match_block in core.cuh); positions are tile positions                  */
template <class C> CLF void t_try_anchor(TileS<C> &T, const TileG<C> &tg, unsigned table, uint32_t i, unsigned pi, uint32_t f) {
    const cl_pattern &p = T.P->pb.p[pi];
    const unsigned nt = p.n_templates;
    const uint32_t b = T.bidx[i], lo = T.bo[b], hi = T.bo[b + 1];
    uint32_t idx[3] = { NONE32, NONE32, NONE32 };
    idx[p.join_order[0]] = i;
    for (unsigned k = 1; k < nt; k++) {
        const unsigned t = p.join_order[k], from = p.join_from[k];
        const cl_hdr hf = T.hdr[idx[from]];
        const cl_template &tf = p.t[from];
        if (hf.n_defs != tf.n_defs || hf.n_aux != tf.n_aux || hf.n_uses != tf.n_uses || (hf.flags & CL_IF_EXT)) return;
        const unsigned long long mm = T.fs.ms[hf.modset].mask;
        if ((mm & tf.mods_all) != tf.mods_all || (mm & tf.mods_none)) return;
        const opnd o = t_slot(T, idx[from], has_guard(hf) + p.join_slot[k]);
        if (!is_value(o)) {
            const unsigned ko = kind_of(o.tag);       /* a non-SSA link: the literal product decides */
            if (ko == CL_K_RZ || ko == CL_K_URZ || ko == CL_K_PRED) tf_fail(T, f, CL_ST_REDO + 1);
            return;
        }
        const uint32_t dp = o.pay < C::V ? T.defpos[o.pay] : NONE32;
        if (dp == NONE32 || dp < lo || dp >= hi || T.hdr[dp].op != p.t[t].op) return;
        idx[t] = dp;
    }
    if (nt > 1 && !(idx[0] < idx[1] && (nt < 3 || idx[1] < idx[2]))) return;
    /* budget (G1): rank of the tuple in itertools.product order, needed only when the
     * product of the candidate-list sizes can exceed it                             */
    {
        uint32_t cn[3] = { 1, 1, 1 };
        int cl[3] = { 0, 0, 0 };
        for (unsigned t = 0; t < nt; t++) { cl[t] = t_class_of(T, table, p.t[t].op); cn[t] = T.ccnt[b][cl[t]]; }
        const unsigned long long prod = (unsigned long long)cn[0] * cn[1] * cn[2];
        if (prod > T.P->pb.budget) {
            unsigned long long r = 0;
            for (unsigned t = 0; t < nt; t++) {
                const uint32_t ci = (uint32_t)T.outpos[idx[t]] - T.cbase[b][cl[t]];      /* index inside its candidate list (t_match) */
                r = t == 0 ? ci : r * cn[t] + ci;
            }
            if (r >= T.P->pb.budget) return;
        }
    }
    if (!t_check_tuple(T, tg, pi, idx)) return;
    const uint32_t m = a_add(&T.n_mt, 1u);
    if (m < C::M) {
        TMatch r;
        r.pat = (uint8_t)pi; r.n = (uint8_t)nt;
        r.pos[0] = (uint16_t)idx[0]; r.pos[1] = (uint16_t)(nt > 1 ? idx[1] : 0xFFFFu); r.pos[2] = (uint16_t)(nt > 2 ? idx[2] : 0xFFFFu);
        T.mt[m] = r;
        T.mstate[m] = MS_UNDECIDED;
    } else
        T.fail = 1;
    a_add(&T.f_stats[f][pi], 1u);
}

/* Counting sort of n work items by pattern (key(k) < CL_MAX_PATTERNS), so that the lanes of a warp run one pattern's
 * code: a histogram and a fill pass, the lanes of a warp that hold the same pattern found by match-any and served by ONE
 * atomic of their leader.  The order inside a pattern is free (matches are keyed, plans are per match); round 1 ran one
 * ordered compaction -- a CTA-wide scan with two barriers per 1024 items -- PER PATTERN here.                    */
template <class G, class C, class FK, class FO> CLD void t_sort_by_pattern(const G &g, TileS<C> &T, uint32_t n, FK key, FO out) {
    GFOR(g, p, CL_MAX_PATTERNS) if (p < CL_MAX_PATTERNS) T.pcnt[p] = 0;
    g.sync();
#if CL_DEV
    auto grouped_add = [&](uint32_t *ctr, unsigned pi) -> uint32_t {      /* slot of this lane among the lanes of its pattern */
        const unsigned peers = __match_any_sync(__activemask(), pi);
        const unsigned lane = threadIdx.x & 31u;
        const int lead = __ffs((int)peers) - 1;
        uint32_t base = 0;
        if ((int)lane == lead) base = atomicAdd(&ctr[pi], (uint32_t)__popc(peers));
        base = __shfl_sync(peers, base, lead);
        return base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
    };
#else
    auto grouped_add = [&](uint32_t *ctr, unsigned pi) -> uint32_t { return ctr[pi]++; };
#endif
    GFOR(g, k, n) if (k < n) grouped_add(T.pcnt, key(k));
    g.sync();
    if (g.rank == 0) { uint32_t run = 0; for (unsigned p = 0; p < CL_MAX_PATTERNS; p++) { T.pcur[p] = run; run += T.pcnt[p]; } }
    g.sync();
    GFOR(g, k, n) if (k < n) out(k, grouped_add(T.pcur, key(k)));
    g.sync();
}

template <class G, class C> CLF void t_match(const G &g, TileS<C> &T, const TileG<C> &tg, unsigned table) {
    PROF(g, T.fs, PF_MATCH);
    GFOR(g, k, T.nb * MAX_CLS) if (k < T.nb * MAX_CLS) (&T.ccnt[0][0])[k] = 0;
    if (g.rank == 0) { T.n_mt = 0; T.n_list = 0; }
    g.sync();
    /* seed classes (FindSeeds) and the dense list of (anchor, pattern) work items, in stream order */
    uint32_t *items = (uint32_t *)T.owner;                   /* [2 * C::I]: free until t_select */
    /* the list of (anchor, pattern) work items; its order is free (the counting sort below groups it by pattern, matches
     * are keyed by position), so a warp reserves room for its items with one atomic: no CTA-wide scan, no barrier */
    GFOR(g, i, T.n) {
        uint32_t pm = 0;
        if (i < T.n) {
            int c = -1;
            const uint32_t f = T.fidx[i];
            if (T.f_gate[f]) {
                c = t_class_of(T, table, T.hdr[i].op);
                if (c >= 0) {
                    a_add(&T.ccnt[T.bidx[i]][c], 1u);
                    if (tf_ok(T, f)) {
                        pm = T.P->anchor_mask[table][c];
                        if (pm && T.f_odd[f]) { tf_fail(T, f, CL_ST_REDO + 2); pm = 0; }
                    }
                }
            }
            T.clsid[i] = (uint8_t)c;
        }
        uint32_t w;
#if CL_DEV
        const uint32_t cnt = (uint32_t)__popc(pm), lane = threadIdx.x & 31u;
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d); if (lane >= (uint32_t)d) incl += t; }
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        uint32_t base = 0;
        if (lane == 31 && tot) base = atomicAdd(&T.n_list, tot);
        base = __shfl_sync(0xFFFFFFFFu, base, 31);
        w = base + incl - cnt;
#else
        uint32_t cnt = 0; for (uint32_t q = pm; q; q &= q - 1) cnt++;
        w = T.n_list; T.n_list += cnt;
#endif
        if (w + cnt <= 2 * C::I) { for (unsigned pi = 0; pm; pi++, pm >>= 1) if (pm & 1u) items[w++] = i | pi << 16; }
        else if (cnt) T.fail = 1;
    }
    g.sync();
    const uint32_t n_items = T.n_list <= 2 * C::I ? T.n_list : 0u;
    g.sync();
    if (T.fail) return;
    /* budget (G1): where the product of the candidate-list sizes of a pattern exceeds it, a tuple counts only
     * if its rank in itertools.product order is below it; the rank needs every member's index inside its
     * candidate list = members of its class before it in the block: one tile-wide scan per class concerned */
    {
        uint32_t need = 0;
        GFOR(g, b, T.nb) if (b < T.nb) {
            uint32_t m = 0;
            for (unsigned pi = 0; pi < T.P->pb.n_patterns; pi++) {
                const cl_pattern &p = T.P->pb.p[pi];
                if (p.table != table) continue;
                unsigned long long prod = 1;
                uint32_t cm = 0;
                for (unsigned t = 0; t < p.n_templates; t++) { const int c = t_class_of(T, table, p.t[t].op); prod *= T.ccnt[b][c]; cm |= 1u << c; }
                if (prod > T.P->pb.budget) m |= cm;
            }
            T.b_over[b] = (uint16_t)m;
            need |= m;
        }
        for (unsigned c = 0; c < T.P->n_cls[table]; c++) {
            if (!g.any((need >> c) & 1u)) continue;
            t_scan(g, T.n, [&](uint32_t j) { return (uint32_t)(T.clsid[j] == c); },
                   [&](uint32_t j, uint32_t x) {
                       if (T.clsid[j] == c) T.outpos[j] = (uint16_t)x;
                       const uint32_t b = T.bidx[j];
                       if (j == T.bo[b]) T.cbase[b][c] = x;
                   });
        }
        g.sync();
    }
    /* the items sorted by pattern (one ordered compaction per pattern of the table), so that the lanes of a warp
     * unify against the same pattern: in stream order neighbouring lanes ran different patterns (2.8 of 32
     * lanes active in the slot tests)                                                                      */
    uint32_t *sorted = (uint32_t *)tg.stage;                 /* free until the rewrites are planned */
    static_assert(sizeof(Stage) * C::S >= 8 * C::I, "staging area holds the sorted work items");
    t_sort_by_pattern(g, T, n_items, [&](uint32_t k) { return items[k] >> 16; }, [&](uint32_t k, uint32_t at) { sorted[at] = items[k]; });
    GFOR(g, k, n_items) if (k < n_items) {
        const uint32_t it = sorted[k], i = it & 0xFFFFu;
        const uint32_t f = T.fidx[i];
        if (tf_ok(T, f)) t_try_anchor(T, tg, table, i, it >> 16, f);
    }
    g.sync();
}

/* select_matches (patterns.py:241-252) for all blocks of the tile at once; the
 * key orders like the reference's stable sort: (start, -len, pattern, product
 * order) where product order within one pattern and start is position order.  */
CLD unsigned long long t_key(const TMatch &m) {
    return (unsigned long long)m.pos[0] << 40 | (unsigned long long)(3u - m.n) << 38 | (unsigned long long)m.pat << 32 |
           (unsigned long long)m.pos[1] << 16 | m.pos[2];
}
template <class G, class C> CLF uint32_t t_select(const G &g, TileS<C> &T) {
    PROF(g, T.fs, PF_SELECT);
    const uint32_t n = T.n, nm = T.n_mt;
    GFOR(g, p, n) if (p < n) { T.keep[p] = 0; T.sel_at[p] = 0xFFFFu; }
    g.sync();
    for (;;) {
        /* only the positions undecided matches still bid for are reset (not every record of the tile) */
        GFOR(g, m, nm) if (m < nm && T.mstate[m] == MS_UNDECIDED) {
            const TMatch r = T.mt[m];
            bool clash = false;
            for (unsigned t = 0; t < r.n; t++) clash |= T.keep[r.pos[t]] != 0;
            if (clash) T.mstate[m] = MS_REJECTED;
            else for (unsigned t = 0; t < r.n; t++) T.owner[r.pos[t]] = NONE64;
        }
        g.sync();
        GFOR(g, m, nm) if (m < nm && T.mstate[m] == MS_UNDECIDED) {
            const TMatch r = T.mt[m];
            const unsigned long long key = t_key(r);
            for (unsigned t = 0; t < r.n; t++) a_min64(&T.owner[r.pos[t]], key);
        }
        g.sync();
        bool left = false;
        GFOR(g, m, nm) if (m < nm && T.mstate[m] == MS_UNDECIDED) {
            const TMatch r = T.mt[m];
            const unsigned long long key = t_key(r);
            bool mine = true;
            for (unsigned t = 0; t < r.n; t++) mine &= T.owner[r.pos[t]] == key;
            if (mine) {
                T.mstate[m] = MS_SELECTED;
                for (unsigned t = 0; t < r.n; t++) T.keep[r.pos[t]] = 1;      /* keep[] is read again only after the sync */
                T.sel_at[r.pos[0]] = (uint16_t)m;
            } else
                left = true;
        }
        const bool again = g.any(left);
        g.sync();
        if (!again) break;
    }
    /* the selected matches in position order (= select order: ids are allocated along it): a scan over contiguous runs */
    uint32_t count = t_scan(g, n, [&](uint32_t p) { return (uint32_t)(T.sel_at[p] != 0xFFFFu); },
                            [&](uint32_t p, uint32_t at) {
                                if (T.sel_at[p] == 0xFFFFu || at >= C::S) return;
                                const TMatch m = T.mt[T.sel_at[p]];
                                SelRec r;
                                r.pat = m.pat; r.n = m.n; r.pad0 = r.pad1 = 0; r.blk = T.bidx[p];
                                r.pos[0] = m.pos[0]; r.pos[1] = m.n > 1 ? m.pos[1] : NONE32; r.pos[2] = m.n > 2 ? m.pos[2] : NONE32;
                                T.sel[at] = r;
                                a_add(&T.f_stats[T.fidx[p]][16 + m.pat], 1u);
                            });
    if (count > C::S) { if (g.rank == 0) T.fail = 1; count = 0; }
    g.sync();
    return count;
}

/* fix-up of one staged match once the bases are known (apply_stage of core.cuh
 * without the in-place retag, which the caller does before the stream moves)   */
template <class C> CLF void t_apply_stage(TileS<C> &T, Stage &st, uint32_t out, uint32_t f, uint32_t blk) {
    for (unsigned k = 0; k < st.nv; k++) {
        const uint32_t v = st.vbase + k;
        if (v >= C::V) continue;
        T.alive[v] = 1; T.origin[v] = CL_ORG_PAIR;
        T.def_iid[v] = st.val_def[k] < 0 ? -1 : (int32_t)(st.ibase + (uint32_t)st.val_def[k]);
    }
    for (unsigned k = 0; k < st.nq; k++) if (st.mbase + k < C::Q) T.imm[st.mbase + k] = st.imm[k];
    if (!st.ok) return;                      /* refused: the allocations above leak (G4) */
    for (unsigned r = 0; r < st.nins; r++) {
        const SRec q = st.rec[r];
        const uint32_t o = out + r;
        cl_hdr h;
        h.iid = st.ibase + q.iid; h.op = q.op; h.modset = q.modset;
        h.n_defs = q.n_defs; h.n_aux = 0; h.n_uses = q.n_uses; h.flags = 0; h.ext = 0;
        T.hdr[o] = h;
        T.fidx[o] = (uint8_t)f; T.bidx[o] = (uint8_t)blk;
        const unsigned ns = (unsigned)q.n_defs + q.n_uses;
#pragma unroll
        for (unsigned k = 0; k < 8; k++) {
            uint16_t tg_ = k < 4 ? q.tag[k] : (uint16_t)0;
            uint32_t py = k < 4 ? q.pay[k] : 0u;
            if (k < ns && (tg_ & CL_T_REL)) {
                py += kind_of(tg_) == CL_K_VALUE ? st.vbase : st.mbase;
                tg_ &= (uint16_t)~CL_T_REL;
            }
            T.tag[(size_t)o * 8 + k] = tg_; T.pay[(size_t)o * 8 + k] = py;
        }
    }
    for (unsigned k = 0; k < st.nupd; k++) if (st.upd_vid[k] < C::V) T.def_iid[st.upd_vid[k]] = (int32_t)(st.ibase + st.upd_iid[k]);
    for (unsigned k = 0; k < st.ndrop; k++) if (st.drop_vid[k] < C::V) T.alive[st.drop_vid[k]] = 0;
}

/* _apply_patterns (patterns.py:671-707): one round over every gated function.
 * All blocks are rewritten against the def-use snapshot of the round's start;
 * a rewrite that removes a use of a value defined in a *later* block of its
 * function would be seen by that block's escape test in the reference (G5):
 * such functions are redone sequentially.                                   */
template <class G, class C> CLF void t_apply_patterns(const G &g, TileS<C> &T, const TileG<C> &tg, unsigned table,
                                                      uint32_t phase) {
    if (!T.du_ok) t_usecount(g, T, tg);
    t_match(g, T, tg, table);
    if (T.fail || T.n_mt == 0) return;
    const uint32_t ns = t_select(g, T);
    if (T.fail || ns == 0) return;
    const uint32_t n = T.n;
    PROF(g, T.fs, PF_PLAN);
    if (T.tombs) { GFOR(g, p, n) if (p < n) { T.keep[p] = T.hdr[p].op != CL_OP_TOMB; T.inscnt[p] = 0; } }     /* the permutation drops them */
    else GFOR(g, p, n) if (p < n) { T.keep[p] = 1; T.inscnt[p] = 0; }
    GFOR(g, f, T.nf) if (f < T.nf) T.f_first[f] = NONE32;
    GFOR(g, b, T.nb) if (b < T.nb) T.b_first[b] = NONE32;
    g.sync();
    /* plan: one lane per selected match, once; lanes take the matches in pattern order (one ordered compaction
     * per pattern), so that a warp runs one rewrite's code: in select order the planners ran at 2-4 active lanes */
    uint32_t *porder = (uint32_t *)T.owner;                  /* free between the selection and the id scans */
    t_sort_by_pattern(g, T, ns, [&](uint32_t j) { return (uint32_t)T.sel[j].pat; }, [&](uint32_t j, uint32_t at) { porder[at] = j; });
    GFOR(g, jq, ns) if (jq < ns) {
        const uint32_t j = porder[jq];
        const SelRec m = T.sel[j];
        Stage &st = tg.stage[j];
        st.ok = st.rm = st.nins = st.retag = st.nv = st.nq = st.nupd = st.ndrop = 0;
        st.ni = 0;
        const uint32_t f = T.fidx[m.pos[0]];
        if (j == 0 || T.fidx[T.sel[j - 1].pos[0]] != f) T.f_first[f] = j;
        if (j == 0 || T.sel[j - 1].blk != m.blk) T.b_first[m.blk] = j;
        if (!tf_ok(T, f)) continue;
        RW c;
        c.s = &T.fs; c.st = &st; c.n = m.n; c.pat = m.pat; c.overflow = false; c.stw = &T.f_stat[f];
        for (unsigned t = 0; t < m.n; t++) { c.idx[t] = m.pos[t]; c.h[t] = T.hdr[c.idx[t]]; }
        for (unsigned t = m.n; t < 3; t++) c.idx[t] = NONE32;
        st.ok = run_rewrite(c);
        if (c.overflow) tf_fail(T, f, CL_ST_REDO + 3);
        if (st.ok && st.rm) {
            /* G5: does a removed record use a value defined in a later block of its function? */
            bool hazard = false;
            for (unsigned t = 0; t < m.n; t++) {
                if (!(st.rm >> t & 1)) continue;
                t_value_operands(T, tg, c.h[t], c.idx[t], [&](uint32_t v) {
                    const uint32_t dp = v < C::V ? T.defpos[v] : NONE32;
                    hazard |= dp != NONE32 && T.bidx[dp] > m.blk;
                });
            }
            if (hazard) tf_fail(T, f, CL_ST_REDO + 4);
        }
    }
    g.sync();
    /* exclusive scans in select order (tile wide; rebased per function below): id bases (G3) */
    t_scan(g, ns, [&](uint32_t j) { const Stage &st = tg.stage[j]; return (uint32_t)st.nv | (uint32_t)st.ni << 16; },
           [&](uint32_t j, uint32_t x) { T.owner[j] = x; });
    t_scan(g, ns, [&](uint32_t j) { return (uint32_t)tg.stage[j].nq; },
           [&](uint32_t j, uint32_t x) { T.owner[j] |= (unsigned long long)x << 32; });
    g.sync();
    GFOR(g, j, ns) if (j < ns) {
        const SelRec m = T.sel[j];
        const uint32_t f = T.fidx[m.pos[0]];
        Stage &st = tg.stage[j];
        const unsigned long long me = T.owner[j], first = T.owner[T.f_first[f]];
        const uint32_t rv = (uint32_t)(me & 0xFFFFu) - (uint32_t)(first & 0xFFFFu);
        const uint32_t ri = (uint32_t)(me >> 16 & 0xFFFFu) - (uint32_t)(first >> 16 & 0xFFFFu);
        const uint32_t rq = (uint32_t)(me >> 32) - (uint32_t)(first >> 32);
        st.vbase = T.f_vbase[f] + T.f_nvid[f] + rv; st.ibase = T.f_niid[f] + ri; st.mbase = T.f_qbase[f] + T.f_nimm[f] + rq;
        if (j + 1 == ns || T.fidx[T.sel[j + 1].pos[0]] != f) {
            /* last match of its function: the function's new counters; over its slices -> general kernel */
            if (st.vbase + st.nv > T.f_vbase[f + 1] || st.mbase + st.nq > T.f_qbase[f + 1]) tf_fail(T, f, CL_ST_REDO + 5);
            T.f_aux[f] = j;
        }
    }
    g.sync();
    GFOR(g, f, T.nf) if (f < T.nf && T.f_first[f] != NONE32 && tf_ok(T, f)) {
        const Stage &st = tg.stage[T.f_aux[f]];
        T.f_nvid[f] = st.vbase + st.nv - T.f_vbase[f]; T.f_niid[f] = st.ibase + st.ni; T.f_nimm[f] = st.mbase + st.nq - T.f_qbase[f];
    }
    /* marks, in-place retags (_rw_imad_wide :414-418), diagnostics, counters */
    GFOR(g, j, ns) if (j < ns) {
        const SelRec m = T.sel[j];
        const uint32_t f = T.fidx[m.pos[0]];
        if (!tf_ok(T, f)) continue;
        Stage &st = tg.stage[j];
        if (st.ok) {
            T.inscnt[m.pos[m.n - 1]] = st.nins;                      /* anchor :689 */
            for (unsigned t = 0; t < m.n; t++) if (st.rm >> t & 1) T.keep[m.pos[t]] = 0;
            if (st.retag) {
                cl_hdr &h = T.hdr[m.pos[0]];
                h.modset = T.fs.ms[h.modset].minus_wide;
                h.op = CL_OP_IMAD64;
            }
            a_add(&T.f_stats[f][32 + m.pat], 1u);
            a_add(&T.f_chg[f], 1u);
        } else {
            a_add(&T.f_stats[f][48 + m.pat], 1u);
            t_event(T, tg, f, phase << 28 | (m.blk - T.f_b0[f]), CL_EV_REFUSED, j - T.b_first[m.blk], m.pat, T.blk[m.blk].bid);
        }
    }
    g.sync();
    /* output position of every record (dead functions keep their records as they are) */
    const uint32_t tot = t_scan(g, n, [&](uint32_t p) { return (uint32_t)T.keep[p] + T.inscnt[p]; },
                                [&](uint32_t p, uint32_t x) { T.outpos[p] = (uint16_t)x; });
    if (tot > C::I) { if (g.rank == 0) T.fail = 1; g.sync(); return; }
    g.sync();
    PROF(g, T.fs, PF_EMIT);
    if constexpr (C::PP) {                 /* def-use of the new stream is taken while it is written (see t_du_record) */
        GFOR(g, v, T.vtot) if (v < T.vtot) { T.usecnt[v] = 0; T.defpos[v] = NONE32; }
        g.sync();
    }
    t_permute<C::PP>(g, T, tg, n, tot, [&](uint32_t p) { return T.keep[p] ? (uint32_t)T.outpos[p] + T.inscnt[p] : NONE32; });
    /* staged records to their place, value table, immediates */
    GFOR(g, j, ns) if (j < ns) {
        const SelRec m = T.sel[j];
        uint32_t f;                                  /* m.pos[] are positions before the permutation */
        if constexpr (C::PP) f = T.fidx.b[m.pos[0]]; else f = T.fidx[m.pos[0]];
        if (!tf_ok(T, f)) continue;
        const uint32_t out0 = T.outpos[m.pos[m.n - 1]];
        t_apply_stage(T, tg.stage[j], out0, f, m.blk);
        if constexpr (C::PP) {
            const Stage &st = tg.stage[j];
            if (st.ok)
                for (unsigned r = 0; r < st.nins; r++) {         /* the records just inserted */
                    const uint32_t o = out0 + r;
                    t_du_record(T, tg, *(const uint4 *)&T.hdr[o], *(const uint4 *)&T.tag[(size_t)o * 8],
                                ((const uint4 *)&T.pay[(size_t)o * 8])[0], ((const uint4 *)&T.pay[(size_t)o * 8])[1], o, f);
                }
        }
    }
    if constexpr (C::PP) {
        GFOR(g, b, T.nb) if (b < T.nb) {                          /* terminator value uses (ssir.py:378-382) */
            if (!tf_ok(T, T.bfun[b])) continue;
            for (int k = 0; k < 2; k++)
                if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE && T.blk[b].term_pay[k] < C::V) a_add(&T.usecnt[T.blk[b].term_pay[k]], 1u);
        }
    }
    g.sync();
    t_rebase_blocks(g, T, n, tot);
    if (g.rank == 0) { T.tombs = 0; if (C::PP) T.du_ok = 1; }
    if constexpr (!C::PP) t_index(g, T);
    /* def-use for simplify_packs / remove_dead_pseudo of this round: taken during the permutation in big tiles,
     * one recount sweep in shared-memory tiles */
    if constexpr (C::PP) g.sync(); else t_usecount(g, T, tg);
}

/* ordered in-place compaction of the stream by keep[]                         */
template <class G, class C> CLF void t_compact(const G &g, TileS<C> &T, const TileG<C> &tg) {
    const uint32_t n = T.n;
    const uint32_t tot = t_scan(g, n, [&](uint32_t p) { return (uint32_t)T.keep[p]; },
                                [&](uint32_t p, uint32_t x) { T.outpos[p] = (uint16_t)x; });
    g.sync();
    t_permute(g, T, tg, n, tot, [&](uint32_t p) { return T.keep[p] ? (uint32_t)T.outpos[p] : NONE32; });
    t_rebase_blocks(g, T, n, tot);
    if constexpr (!C::PP) t_index(g, T);
}

/* remove_dead_pseudo (patterns.py:771-791) for the functions with f_gate set.  The first sweep visits the
 * records; pure records that survive it are the only ones that can still die: the later rounds of the
 * fixpoint walk that list                                                                               */
template <class G, class C> CLF void t_dce(const G &g, TileS<C> &T, const TileG<C> &tg) {
    PROF(g, T.fs, PF_DCE);
    if (!T.du_ok) t_usecount(g, T, tg);
    uint32_t *list = (uint32_t *)T.owner;                 /* [<= I] */
    if (g.rank == 0) T.n_list = 0;
    g.sync();
    auto try_kill = [&](uint32_t i, const cl_hdr &h) -> bool {
        unsigned nd = 0; bool used = false;
        t_value_defs(T, h, i, [&](uint32_t v) { nd++; used |= v < C::V && *(volatile uint32_t *)&T.usecnt[v] != 0; });
        if (!nd) return true;                               /* never dies: not a candidate either */
        if (used) return false;
        T.keep[i] = 0;
        t_value_defs(T, h, i, [&](uint32_t v) { if (v < C::V) T.alive[v] = 0; });
        t_value_operands(T, tg, h, i, [&](uint32_t v) { if (v < C::V) a_sub(&T.usecnt[v], 1u); });
        return true;
    };
    uint32_t mine = 0;
    GFOR(g, i, T.n) if (i < T.n) {
        T.keep[i] = 1;
        const uint32_t f = T.fidx[i];
        if (!T.f_gate[f] || !tf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        if (h.op >= CL_OP__COUNT || !(T.fs.opflags[h.op] & CL_OPF_PURE)) continue;
        if (try_kill(i, h)) mine += T.keep[i] == 0;
        else list[a_add(&T.n_list, 1u)] = i;
    }
    uint32_t removed = 0;
    for (;;) {
        const uint32_t dead = g.sum(mine);
        g.sync();
        if (!dead) break;
        removed += dead;
        mine = 0;
        const uint32_t nl = T.n_list;
        GFOR(g, k, nl) if (k < nl) {
            const uint32_t i = list[k];
            if (!T.keep[i] || !tf_ok(T, T.fidx[i])) continue;
            if (try_kill(i, T.hdr[i])) mine++;
        }
    }
    if (removed) {
        GFOR(g, i, T.n) if (i < T.n && !T.keep[i]) {
            cl_hdr h = T.hdr[i];
            h.op = CL_OP_TOMB; h.modset = 0; h.n_defs = h.n_aux = h.n_uses = 0; h.flags = 0; h.ext = 0;
            T.hdr[i] = h;
        }
        if (g.rank == 0) T.tombs = 1;
        g.sync();
    }
}

/* simplify_packs + _redirect_values (patterns.py:710-764) for the gated functions;
 * f_red[f] = redirects of function f                                          */
template <class C> CLD uint32_t t_final_of(const TileS<C> &T, uint32_t v) {
    while (v < C::V && T.redirect[v] != NONE32) v = T.redirect[v];
    return v;
}
template <class G, class C> CLF void t_simplify(const G &g, TileS<C> &T, const TileG<C> &tg) {
    PROF(g, T.fs, PF_SIMPLIFY);
    const FS &s = T.fs;
    if (!T.du_ok) t_usecount(g, T, tg);
    GFOR(g, v, T.vtot) if (v < T.vtot) T.redirect[v] = NONE32;
    GFOR(g, f, T.nf) if (f < T.nf) T.f_red[f] = 0;
    g.sync();
    uint32_t mine = 0;
    GFOR(g, i, T.n) if (i < T.n) {
        const cl_hdr h = T.hdr[i];
        if (h.op != CL_OP_PACK64 || h.n_uses != 2) continue;
        const uint32_t f = T.fidx[i];
        if (!T.f_gate[f] || !tf_ok(T, f)) continue;
        const unsigned u0 = use0(h);
        const opnd lo = t_slot(T, i, u0), hi = t_slot(T, i, u0 + 1);
        if (!is_value(lo) || !is_value(hi)) continue;
        if ((lo.tag | hi.tag) & (CL_T_NEG | CL_T_NOT)) continue;
        if (lo.pay >= C::V || hi.pay >= C::V) continue;
        const uint32_t plo = T.defpos[lo.pay], phi = T.defpos[hi.pay];
        if (plo == NONE32 || phi == NONE32) continue;
        const cl_hdr dlo = T.hdr[plo], dhi = T.hdr[phi];
        if (!(dlo.op == CL_OP_UNPACK64 && has_mod(s, dlo, CL_MB_LO) && dhi.op == CL_OP_UNPACK64 && has_mod(s, dhi, CL_MB_HI))) continue;
        if (!dlo.n_uses || !dhi.n_uses) { tf_fail(T, f, CL_ST_REDO + 6); continue; }
        const opnd slo = t_slot(T, plo, use0(dlo)), shi = t_slot(T, phi, use0(dhi));
        if (!(is_value(slo) && is_value(shi) && slo.pay == shi.pay)) continue;
        if (!h.n_defs) { tf_fail(T, f, CL_ST_REDO + 7); continue; }
        const opnd d = t_slot(T, i, def0(h));
        if (!is_value(d)) { tf_fail(T, f, CL_ST_REDO + 8); continue; }
        if (d.pay < C::V) T.redirect[d.pay] = slo.pay;
        a_add(&T.f_red[f], 1u);
        mine++;
    }
    const uint32_t changed = g.sum(mine);
    g.sync();
    if (!changed) return;
    /* the use counts follow the redirects (every use site of the old value becomes one of the new) */
    auto move_use = [&](uint32_t v) {
        const uint32_t fo = t_final_of(T, v);
        if (fo != v && v < C::V) { a_sub(&T.usecnt[v], 1u); if (fo < C::V) a_add(&T.usecnt[fo], 1u); }
    };
    GFOR(g, i, T.n) if (i < T.n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_red[f] || !tf_ok(T, f)) continue;
        t_value_operands(T, tg, T.hdr[i], i, move_use);
    }
    GFOR(g, b, T.nb) if (b < T.nb) {
        const uint32_t f = T.bfun[b];
        if (!T.f_red[f] || !tf_ok(T, f)) continue;
        for (int k = 0; k < 2; k++) if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE) move_use(T.blk[b].term_pay[k]);
    }
    g.sync();
    GFOR(g, i, T.n) if (i < T.n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_red[f] || !tf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) {
            const opnd u = t_slot(T, i, u0 + k);
            if (is_value(u)) { const uint32_t fo = t_final_of(T, u.pay); if (fo != u.pay) T.pay[(size_t)i * 8 + u0 + k] = fo; }
            else if (kind_of(u.tag) == CL_K_MEMREF) {
                cl_memref &m = tg.mem[u.pay];
                if (kind_of(m.base_tag) == CL_K_VALUE) m.base_pay = t_final_of(T, m.base_pay);
                if (kind_of(m.ureg_tag) == CL_K_VALUE) m.ureg_pay = t_final_of(T, m.ureg_pay);
            }
        }
        if (has_guard(h)) { const opnd gd = t_slot(T, i, 0); if (is_value(gd)) T.pay[(size_t)i * 8] = t_final_of(T, gd.pay); }
    }
    GFOR(g, b, T.nb) if (b < T.nb) {
        const uint32_t f = T.bfun[b];
        if (!T.f_red[f] || !tf_ok(T, f)) continue;
        for (int k = 0; k < 2; k++)
            if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE) T.blk[b].term_pay[k] = t_final_of(T, T.blk[b].term_pay[k]);
    }
    g.sync();
}

/* tag_cuda_objects (patterns.py:895-916)                                      */
template <class G, class C> CLF void t_tag(const G &g, TileS<C> &T) {
    PROF(g, T.fs, PF_TAG);
    const FS &s = T.fs;
    GFOR(g, i, T.n) if (i < T.n) {
        cl_hdr h = T.hdr[i];
        if (h.op != CL_OP_BAR && h.op != CL_OP_WARPSYNC && h.op != CL_OP_SHFL) continue;
        if (!tf_ok(T, T.fidx[i])) continue;
        unsigned kind = 0, use = 7;
        const unsigned u0 = use0(h);
        if (h.op == CL_OP_BAR) {
            if (has_mod(s, h, CL_MB_SYNC)) {
                kind = 1;
                for (unsigned k = 0; k < h.n_uses && k < 7; k++) if (is_imm(t_slot(T, i, u0 + k))) use = k;
            }
        } else if (h.op == CL_OP_WARPSYNC) {
            for (unsigned k = 0; k < h.n_uses && k < 7; k++) {
                const opnd u = t_slot(T, i, u0 + k);
                if (is_imm(u)) { if (T.imm[u.pay].bits == 0xFFFFFFFFull) { kind = 2; use = k; } break; }
            }
        } else
            kind = 3;
        if (kind) {
            h.flags &= (uint8_t)~(CL_IF_OBJ_MASK | CL_IF_OBJUSE_MASK);
            h.flags |= (uint8_t)(kind << CL_IF_OBJ_SHIFT | use << CL_IF_OBJUSE_SHIFT);
            T.hdr[i].flags = h.flags;
        }
    }
    g.sync();
}

/* ------------------------------------------------------- reciprocal chains */
/* normalize_reciprocal (patterns.py:817-888), chains in parallel.
 *   R_k(r): an F2I is reachable from record r in <= k def-use hops (_reaches_f2i :850)
 *           -- backward propagation from the F2I records, three sweeps;
 *   a chain (MUFU.RCP of an I2F, IADD/IADD3 with an immediate using it) is
 *   accepted iff R_3(add);
 *   its number (vids, iids, boundary index) is its rank by (mufu, add) position.
 * The reference rewrites chain after chain on a rebuilt def-use graph; a later
 * chain sees an earlier one only if its search walks over that chain's add or
 * MUFU.  Functions where an accepted add reaches another accepted chain within
 * two hops, adds with two reciprocal operands and every exception path of the
 * reference are redone by the sequential kernel.                            */
enum { RF_R0 = 1, RF_R1 = 2, RF_R2 = 4, RF_R3 = 8, RF_SEED = 16, RF_Q = 32, RF_MUFU = 128 };
/* one byte of a per-record flag array (4-byte aligned) as an atomic OR; returns the byte before */
CLD uint32_t t_flag_or(uint8_t *flags, uint32_t i, uint32_t bits) {
    const uint32_t sh = (i & 3u) * 8u;
    return (a_or((uint32_t *)flags + (i >> 2), bits << sh) >> sh) & 0xFFu;
}
/* backward propagation of "an F2I is reachable in <= k hops" over the def-use graph, level by level on work
 * lists: W[w0, w1) holds the records that became reachable at the level before; the defining record of every
 * value such a record reads becomes reachable one hop later.  Work is proportional to the cones of the F2I
 * records, not to the tile.  `blocked`: records with RF_SEED in T.flag pass nothing on (paths through them
 * do not count).  Returns the end of the list.                                                          */
template <class G, class C> CLD uint32_t t_reach_levels(const G &g, TileS<C> &T, const TileG<C> &tg, uint8_t *fl, uint32_t *W,
                                                        uint32_t w0, uint32_t w1, bool blocked) {
    for (unsigned k = 1; k <= 3; k++) {
        const uint32_t bits = (0xFu << k) & 0xFu, bit = 1u << k;
        GFOR(g, q, w1 - w0) if (q < w1 - w0) {
            const uint32_t i = W[w0 + q], f = T.fidx[i];
            if (!T.f_rgate[f] || !tf_ok(T, f)) continue;
            if (blocked && (T.flag[i] & RF_SEED)) continue;
            t_value_operands(T, tg, T.hdr[i], i, [&](uint32_t v) {
                const uint32_t dp = v < C::V ? T.defpos[v] : NONE32;
                if (dp == NONE32 || (fl[dp] & bit)) return;
                const uint32_t before = t_flag_or(fl, dp, bits);
                if (!(before & bit) && k < 3) W[a_append(&T.n_list)] = dp;      /* first to reach it */
            });
        }
        g.sync();
        w0 = w1; w1 = T.n_list;
        g.sync();
        if (w1 == w0) break;
    }
    return w1;
}
/* The chains the two propagations leave undecided (an F2I within three hops, but only on paths through other
 * chains), decided exactly and in the reference's order (MUFU position, then add position).  What an accepted
 * chain A changes for a later one (_insert_reciprocal_bitcasts, patterns.py:863-888): the result of its add is
 * read through the new BITCAST.I2F by every top-level use (guards and address bases keep reading it directly),
 * and its add reads the MUFU result through the new BITCAST.F2I: those def-use edges count two hops.  Chain B
 * is accepted iff an F2I lies within weighted distance three of its add, with the chains accepted before it as
 * the two-hop edges: three sweeps over the function's records per chain (cost 0, 1, 2 frontiers), whole CTA.
 * Rejected chains leave the list; returns its new length.                                                 */
static constexpr uint32_t T_MAX_UNDECIDED = 32;
template <class G, class C> CLF uint32_t t_decide_chains(const G &g, TileS<C> &T, const TileG<C> &tg, uint32_t *ul, uint32_t n_u,
                                                         uint32_t nc, uint8_t *cost) {
    uint32_t *vcost = T.redirect;                        /* [V] cost of the record defining the value, NONE32 = not reached */
    uint16_t *chain_of = T.sel_at;                       /* [I] chain whose add the record is, 0xFFFF = none */
    auto key_of = [&](const TChain &c) { return (uint32_t)c.mufu << 16 | c.add; };
    GFOR(g, i, T.n) if (i < T.n) chain_of[i] = 0xFFFFu;
    g.sync();
    GFOR(g, c, nc) if (c < nc) { TChain &ch = T.chain[c]; chain_of[ch.add] = (uint16_t)c; ch.ok = (T.flag[ch.add] & RF_Q) ? 2 : 1; }
    if (g.rank == 0)                                     /* a handful: insertion sort by chain order */
        for (uint32_t a = 1; a < n_u; a++) {
            const uint32_t x = ul[a]; uint32_t b = a;
            while (b > 0 && key_of(T.chain[ul[b - 1]]) > key_of(T.chain[x])) { ul[b] = ul[b - 1]; b--; }
            ul[b] = x;
        }
    g.sync();
    for (uint32_t q = 0; q < n_u; q++) {
        const uint32_t cb = ul[q];
        const TChain B = T.chain[cb];
        const uint32_t f = B.f, kb = key_of(B);
        if (!tf_ok(T, f)) continue;                      /* uniform: every lane reads the same word after the sync */
        const uint32_t i0 = T.bo[T.f_b0[f]], i1 = T.bo[T.f_b0[f + 1]], v0 = T.f_vbase[f], v1 = T.f_vbase[f + 1];
        GFOR(g, v, v1 - v0) if (v < v1 - v0) vcost[v0 + v] = NONE32;
        GFOR(g, i, i1 - i0) if (i < i1 - i0) cost[i0 + i] = 0xFF;
        if (g.rank == 0) T.work = 0;
        g.sync();
        if (g.rank == 0) cost[B.add] = 0;
        g.sync();
        for (uint32_t c = 0; c < 3; c++) {
            GFOR(g, i, i1 - i0) if (i < i1 - i0 && cost[i0 + i] == c)
                t_value_defs(T, T.hdr[i0 + i], i0 + i, [&](uint32_t v) { if (v < C::V) vcost[v] = c; });
            g.sync();
            GFOR(g, ii, i1 - i0) if (ii < i1 - i0) {
                const uint32_t u = i0 + ii;
                const cl_hdr h = T.hdr[u];
                uint32_t best = 0xFF;
                auto edge = [&](uint32_t v, bool top) {
                    if (v >= C::V || vcost[v] != c) return;
                    const uint32_t r = T.defpos[v];
                    uint32_t w = 1;
                    if (r != NONE32 && top) {
                        const uint32_t ca = chain_of[r];           /* r is the add of an accepted earlier chain */
                        if (ca != 0xFFFFu && T.chain[ca].ok == 1 && key_of(T.chain[ca]) < kb) w = 2;
                        const uint32_t cu = chain_of[u];           /* u is the add of one, reading its MUFU's result */
                        if (cu != 0xFFFFu && T.chain[cu].ok == 1 && key_of(T.chain[cu]) < kb && T.chain[cu].mufu == r && T.chain[cu].rcp == v) w = 2;
                    }
                    if (c + w < best) best = c + w;
                };
                if (has_guard(h)) { const opnd gd = t_slot(T, u, 0); if (is_value(gd)) edge(gd.pay, false); }
                const unsigned u0 = use0(h);
                for (unsigned k = 0; k < h.n_uses; k++) {
                    const opnd x = t_slot(T, u, u0 + k);
                    if (is_value(x)) edge(x.pay, true);
                    else if (kind_of(x.tag) == CL_K_MEMREF) {
                        const cl_memref &m = tg.mem[x.pay];
                        if (kind_of(m.base_tag) == CL_K_VALUE) edge(m.base_pay, false);
                        if (kind_of(m.ureg_tag) == CL_K_VALUE) edge(m.ureg_pay, false);
                    }
                }
                if (best <= 3) {
                    if (h.op == CL_OP_F2I) T.work = 1;
                    else if (best < cost[u]) cost[u] = (uint8_t)best;
                }
            }
            g.sync();
        }
        if (g.rank == 0) { T.chain[cb].ok = T.work ? 1 : 0; T.flag[B.add] &= (uint8_t)~RF_Q; }
        g.sync();
    }
    /* rejected chains leave the list (ordered compaction by one lane: the list is short work next to the sweeps) */
    if (g.rank == 0) {
        uint32_t w = 0;
        for (uint32_t c = 0; c < nc; c++) {
            const TChain ch = T.chain[c];
            if (ch.ok == 0) { T.f_aux[ch.f]--; T.flag[ch.add] &= (uint8_t)~RF_SEED; continue; }
            T.chain[w] = ch; T.chain[w].ok = 1; w++;
        }
        T.n_chain = w;
    }
    g.sync();
    return T.n_chain;
}
template <class G, class C> CLF void t_reciprocal(const G &g, TileS<C> &T, const TileG<C> &tg) {
    PROF(g, T.fs, PF_RECIP);
    const FS &s = T.fs;
    if (!T.du_ok) t_usecount(g, T, tg);
    const uint32_t n = T.n;
    uint32_t *W = (uint32_t *)T.owner;                    /* [2 I] work lists (every record enters at most once per propagation) */
    uint16_t *cands = T.outpos;                           /* [I] IADD / IADD3 records, candidates for the add of a chain          */
    uint8_t *fl2 = T.clsid;                               /* [I] reach flags of the propagation that avoids the chain records    */
    GFOR(g, f, T.nf) if (f < T.nf) T.f_aux[f] = 0;
    if (g.rank == 0) { T.n_chain = 0; T.n_list = 0; T.work = 0; }
    g.sync();
    /* one sweep: R_0 (the F2I records, start of the work list), the MUFU.RCP records fed by an I2F (only functions
     * holding one take part: f_rgate, cleared by t_load), the IADD / IADD3 records                                   */
    bool mine = false;
    GFOR(g, i, n) if (i < n) {
        const uint32_t f = T.fidx[i];
        const cl_hdr h = T.hdr[i];
        uint8_t fl = 0;
        if (h.op == CL_OP_F2I) { fl = (uint8_t)(RF_R0 | RF_R1 | RF_R2 | RF_R3); W[a_append(&T.n_list)] = i; }
        else if (h.op == CL_OP_IADD || h.op == CL_OP_IADD3) cands[a_append(&T.work)] = (uint16_t)i;
        else if (h.op == CL_OP_MUFU && has_mod(s, h, CL_MB_RCP)) {
            T.f_rgate[f] = 1;
            if (tf_ok(T, f) && h.n_uses) {
                const opnd src = t_slot(T, i, use0(h));
                if (is_value(src) && src.pay < C::V) {
                    const uint32_t dp = T.defpos[src.pay];
                    if (dp != NONE32 && T.hdr[dp].op == CL_OP_I2F) {
                        if (!h.n_defs || !is_value(t_slot(T, i, def0(h)))) tf_fail(T, f, CL_ST_REDO + 9);   /* IndexError / AttributeError */
                        else { fl |= RF_MUFU; mine = true; }
                    }
                }
            }
        }
        T.flag[i] = fl; fl2[i] = fl & 0xFu;
    }
    if (!g.any(mine)) return;
    g.sync();
    const uint32_t n_f2i = T.n_list, n_cand = T.work;
    g.sync();
    uint32_t w_end = t_reach_levels(g, T, tg, T.flag, W, 0, n_f2i, false);
    /* accepted chains */
    GFOR(g, q, n_cand) if (q < n_cand) {
        const uint32_t i = cands[q], f = T.fidx[i];
        if (!T.f_rgate[f] || !tf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        bool any_imm = false;
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) any_imm |= is_imm(t_slot(T, i, u0 + k));
        if (!any_imm) continue;
        unsigned hits = 0;
        uint32_t mp = NONE32, rcp = 0;
        t_value_operands(T, tg, h, i, [&](uint32_t v) {
            const uint32_t dp = v < C::V ? T.defpos[v] : NONE32;
            if (dp == NONE32 || !(T.flag[dp] & RF_MUFU)) return;
            const opnd d0 = t_slot(T, dp, def0(T.hdr[dp]));
            if (!is_value(d0) || d0.pay != v) return;
            hits++; mp = dp; rcp = v;
        });
        if (!hits) continue;
        if (!(T.flag[i] & RF_R3)) continue;          /* no F2I within three hops before any rewrite, none after: rewrites only lengthen paths */
        if (hits > 1 || has_guard(h) || (h.flags & CL_IF_EXT)) { tf_fail(T, f, CL_ST_REDO + 10); continue; }
        if (T.bidx[mp] != T.bidx[i] || !h.n_defs || !is_value(t_slot(T, i, def0(h)))) { tf_fail(T, f, CL_ST_REDO + 11); continue; }
        const uint32_t c = a_add(&T.n_chain, 1u);
        if (c < C::X) {
            TChain ch;
            ch.add = (uint16_t)i; ch.mufu = (uint16_t)mp; ch.rcp = rcp; ch.addv = t_slot(T, i, def0(h)).pay; ch.f = (uint8_t)f; ch.ok = 1; ch.rank = 0;
            T.chain[c] = ch;
        } else
            T.fail = 1;
        t_flag_or(T.flag, i, RF_SEED);
        t_flag_or(T.flag, mp, RF_SEED);
        a_add(&T.f_aux[f], 1u);
    }
    g.sync();
    uint32_t nc = T.n_chain;
    if (nc == 0 || T.fail) return;
    /* interference.  The reference rewrites chain after chain on a rebuilt def-use graph, and a rewritten chain
     * lengthens by one hop every path through the result of its add or of its MUFU.  A chain whose add reaches an
     * F2I within three hops on a path that passes through NO record of an accepted chain (its own add is the
     * start, not a passage) is accepted whatever was rewritten before it: reach flags of a second propagation in
     * which the chain records pass nothing on (functions with one chain need none).  A chain that reaches its F2I
     * only through other chains depends on their order: the function is redone by the sequential kernel.      */
    bool multi = false;
    uint32_t nc_final = nc;
    GFOR(g, f, T.nf) if (f < T.nf) multi |= T.f_aux[f] > 1;
    if (g.any(multi)) {
        if (w_end + n_f2i > 2 * C::I) { if (g.rank == 0) T.fail = 1; g.sync(); return; }
        GFOR(g, q, n_f2i) if (q < n_f2i) W[w_end + q] = W[q];
        if (g.rank == 0) T.n_list = w_end + n_f2i;
        g.sync();
        t_reach_levels(g, T, tg, fl2, W, w_end, w_end + n_f2i, true);
        if (g.rank == 0) T.n_list = 0;
        g.sync();
        uint32_t *ul = W;                                     /* the undecided chains (the work lists are done) */
        GFOR(g, c, nc) if (c < nc) {
            const TChain ch = T.chain[c];
            if (T.f_aux[ch.f] > 1 && !(fl2[ch.add] & RF_R3) && tf_ok(T, ch.f)) { T.flag[ch.add] |= RF_Q; ul[a_append(&T.n_list)] = c; }
        }
        g.sync();
        const uint32_t n_u = T.n_list;
#if !CL_DEV
        if (n_u && getenv("CL_DEBUG_REDO")) fprintf(stderr, "tile reciprocal: %u chain(s) of %u undecided by the propagations\n", n_u, nc);
#endif
        if (n_u && n_u <= T_MAX_UNDECIDED) nc_final = t_decide_chains(g, T, tg, ul, n_u, nc, fl2);
    }
    nc = nc_final;
    GFOR(g, i, n) if (i < n) { T.keep[i] = 0; T.inscnt[i] = 0; }
    /* rank, ids, value table; vmap (usecnt[]) = add result -> its float view */
    GFOR(g, v, T.vtot) if (v < T.vtot) T.usecnt[v] = NONE32;
    g.sync();
    /* number of a chain inside its function = chains of earlier MUFUs (scan over the records) + chains of
     * the same MUFU with an earlier add (a short list per MUFU: owner[m] low word = head, TChain.rank = next) */
    GFOR(g, i, n) if (i < n && T.f_rgate[T.fidx[i]]) T.owner[i] = 0xFFFFFFFFull;   /* high word: chains of this MUFU */
    g.sync();
    GFOR(g, c, nc) if (c < nc) {
        TChain &ch = T.chain[c];
        if ((T.flag[ch.add] & RF_Q) != 0) { tf_fail(T, ch.f, CL_ST_REDO + 12); continue; }
#if CL_DEV
        ch.rank = (uint16_t)atomicExch((uint32_t *)&T.owner[ch.mufu], c);
        atomicAdd((uint32_t *)&T.owner[ch.mufu] + 1, 1u);
#else
        ch.rank = (uint16_t)(uint32_t)T.owner[ch.mufu];
        T.owner[ch.mufu] = ((T.owner[ch.mufu] >> 32) + 1) << 32 | c;
#endif
    }
    g.sync();
    t_scan(g, n, [&](uint32_t j) { return T.f_rgate[T.fidx[j]] ? (uint32_t)(T.owner[j] >> 32) : 0u; },
           [&](uint32_t j, uint32_t x) {
               T.outpos[j] = (uint16_t)x;
               const uint32_t f = T.fidx[j];
               if (j == T.bo[T.f_b0[f]]) T.f_first[f] = x;
           });
    g.sync();
    GFOR(g, c, nc) if (c < nc) {
        const TChain ch = T.chain[c];
        if (!tf_ok(T, ch.f)) continue;
        uint32_t within = 0;
        for (uint32_t o = (uint32_t)T.owner[ch.mufu] & 0xFFFFu; o != 0xFFFFu; o = T.chain[o].rank)
            within += T.chain[o].add < ch.add;
        T.sel_at[ch.add] = (uint16_t)((uint32_t)T.outpos[ch.mufu] - T.f_first[ch.f] + within);
    }
    g.sync();
    GFOR(g, c, nc) if (c < nc) { TChain &ch = T.chain[c]; if (tf_ok(T, ch.f)) ch.rank = T.sel_at[ch.add]; }
    g.sync();
    GFOR(g, c, nc) if (c < nc) {
        const TChain ch = T.chain[c];
        const uint32_t f = ch.f;
        if (!tf_ok(T, f)) continue;
        const uint32_t vb = T.f_vbase[f];
        const uint32_t vi = vb + T.f_nvid[f] + 2u * ch.rank, vf = vi + 1u, iid = T.f_niid[f] + 2u * ch.rank;
        if (vf >= T.f_vbase[f + 1]) { tf_fail(T, f, CL_ST_REDO + 13); continue; }
        /* _insert_reciprocal_bitcasts :863-888 (origin codes carry function-local vids) */
        T.alive[vi] = 1; T.origin[vi] = CL_ORG_BITS | (ch.rcp - vb); T.def_iid[vi] = (int32_t)iid;
        T.alive[vf] = 1; T.origin[vf] = CL_ORG_F | (ch.addv - vb); T.def_iid[vf] = (int32_t)(iid + 1u);
        const cl_hdr ah = T.hdr[ch.add];
        const unsigned u0 = use0(ah);
        for (unsigned k = 0; k < ah.n_uses; k++) {
            const opnd x = t_slot(T, ch.add, u0 + k);
            if (is_value(x) && x.pay == ch.rcp) T.pay[(size_t)ch.add * 8 + u0 + k] = vi;
        }
        T.usecnt[ch.addv] = vf;
        T.keep[ch.add] = 1; T.inscnt[ch.add] = 1;
        t_event(T, tg, f, 1u << 28, CL_EV_BOUNDARY, ch.rank, ch.rcp - vb, ah.iid);
    }
    g.sync();
    /* every user of an add result (top-level uses only :878-883) reads the float view */
    GFOR(g, i, n) if (i < n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_aux[f] || !tf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) {
            const opnd x = t_slot(T, i, u0 + k);
            if (is_value(x) && x.pay < C::V && T.usecnt[x.pay] != NONE32) T.pay[(size_t)i * 8 + u0 + k] = T.usecnt[x.pay];
        }
    }
    g.sync();
    /* materialise the bitcasts */
    const uint32_t tot = t_scan(g, n, [&](uint32_t p) { return 1u + T.keep[p] + T.inscnt[p]; },
                                [&](uint32_t p, uint32_t x) { T.outpos[p] = (uint16_t)x; });
    if (tot > C::I) { if (g.rank == 0) T.fail = 1; g.sync(); return; }
    g.sync();
    if constexpr (C::PP) {                 /* usecnt[] was the float-view map until here; now the def-use of the new stream */
        GFOR(g, v, T.vtot) if (v < T.vtot) { T.usecnt[v] = 0; T.defpos[v] = NONE32; }
        g.sync();
    }
    t_permute<C::PP>(g, T, tg, n, tot, [&](uint32_t p) { return (uint32_t)T.outpos[p] + T.keep[p]; });
    GFOR(g, c, nc) if (c < nc) {
        const TChain ch = T.chain[c];
        const uint32_t f = ch.f;
        if (!tf_ok(T, f)) continue;
        const uint32_t vi = T.f_vbase[f] + T.f_nvid[f] + 2u * ch.rank, iid = T.f_niid[f] + 2u * ch.rank;
        for (unsigned q = 0; q < 2; q++) {
            const uint32_t o = (uint32_t)T.outpos[ch.add] + 2u * q;
            cl_hdr h;
            h.iid = iid + q; h.op = CL_OP_BITCAST; h.modset = q ? CL_MS_I2F : CL_MS_F2I;
            h.n_defs = 1; h.n_aux = 0; h.n_uses = 1; h.flags = 0; h.ext = 0;
            T.hdr[o] = h;
            T.fidx[o] = (uint8_t)f; T.bidx[o] = T.bidx[(uint32_t)T.outpos[ch.add] + 1u];      /* the add itself sits between the two */
            for (unsigned k = 0; k < 8; k++) { T.tag[(size_t)o * 8 + k] = k < 2 ? (uint16_t)CL_K_VALUE : (uint16_t)0; T.pay[(size_t)o * 8 + k] = 0; }
            T.pay[(size_t)o * 8] = vi + q; T.pay[(size_t)o * 8 + 1] = q ? ch.addv : ch.rcp;
            if constexpr (C::PP) {
                if (vi + q < C::V) T.defpos[vi + q] = o;
                const uint32_t src = q ? ch.addv : ch.rcp;
                if (src < C::V) a_add(&T.usecnt[src], 1u);
            }
        }
    }
    if constexpr (C::PP) {
        GFOR(g, b, T.nb) if (b < T.nb) {                          /* terminator value uses (ssir.py:378-382) */
            if (!tf_ok(T, T.bfun[b])) continue;
            for (int k = 0; k < 2; k++)
                if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE && T.blk[b].term_pay[k] < C::V) a_add(&T.usecnt[T.blk[b].term_pay[k]], 1u);
        }
    }
    g.sync();
    GFOR(g, f, T.nf) if (f < T.nf && T.f_aux[f] && tf_ok(T, f)) { T.f_nvid[f] += 2u * T.f_aux[f]; T.f_niid[f] += 2u * T.f_aux[f]; }
    t_rebase_blocks(g, T, n, tot);
    if constexpr (C::PP) { if (g.rank == 0) T.du_ok = 1; g.sync(); } else t_index(g, T);
}

/* ------------------------------------------------------------ load / store */
/* capacities a function gets inside a tile (host planner and device agree)    */
CLHD uint32_t tile_icap(uint32_t nrec) { return nrec + nrec / 2 + 8; }
CLHD uint32_t tile_vcap(uint32_t nvid, uint32_t nrec) { return nvid + nrec + 8; }
/* new immediates: the growth allowance flattens above 512 records (a 9 600-record block fits the 5 120 of a big
 * tile); an overflow of the slice is detected and the function redone by the general kernel                    */
CLHD uint32_t tile_qcap(uint32_t nimm, uint32_t nrec) { return nimm + (nrec <= 512 ? nrec / 2 : 256 + (nrec - 512) / 8) + 8; }

struct TileIO {                /* the part of KArgs the tile kernel needs (see culifter.cu) */
    cl_corpus in;
    cl_hdr *o_hdr; uint16_t *o_tag; uint32_t *o_pay; cl_imm *o_imm;
    uint8_t *o_alive; int32_t *o_def_iid; uint32_t *o_origin;
    cl_memref *o_mem;
    cl_blk *o_blk; uint32_t *o_blk_start, *o_blk_cnt;
    cl_event *o_ev;
    void *o_func;              /* FuncOut[]                                       */
    unsigned long long cap[4];
    unsigned long long *cursor, *stats;
    uint32_t *retry_list, *retry_count;
    uint32_t *retry_big_list, *retry_big_count; uint32_t small_max;
    const uint32_t *flist;     /* function ids of all tiles                          */
};
struct TFuncOut { cl_func f; uint32_t inst_start, n_inst, imm_start, n_imm, val_start, ev_start, n_ev, pad; };

/* slice that holds tile index k: last f with base[f] <= k                      */
CLD uint32_t t_slice_of(const uint32_t *base, uint32_t nf, uint32_t k) {
    uint32_t lo = 0, hi = nf;
    while (lo + 1 < hi) { const uint32_t mid = (lo + hi) >> 1; if (base[mid] <= k) lo = mid; else hi = mid; }
    return lo;
}
/* rebase the ids of one operand into (in) or out of the tile's index spaces    */
template <class C> CLD uint32_t t_rebase(const TileS<C> &T, uint32_t f, uint16_t tag, uint32_t pay, bool in) {
    uint32_t d;
    switch (kind_of(tag)) {
    case CL_K_VALUE: d = T.f_vbase[f]; break;
    case CL_K_IMM: d = T.f_qbase[f]; break;
    case CL_K_MEMREF: d = T.f_mbase[f]; break;
    default: return pay;
    }
    return in ? pay + d : pay - d;
}

template <class G, class C> CLF void t_load(const G &g, TileS<C> &T, TileG<C> &tg, const TileIO &a, const TileDesc td) {
    PROF(g, T.fs, PF_LOAD);
    const cl_corpus &in = a.in;
    const uint32_t nf = td.nf;
    tg.mem = a.o_mem;
    if (g.rank == 0) {
        T.fs.mem = tg.mem;
        T.nf = nf;
        T.n_ev = 0; T.fail = 0; T.n_chain = 0; T.n_mt = 0; T.n_sel = 0; T.du_ok = 0; T.n_list = 0; T.tombs = 0;
    }
    GFOR(g, f, nf) if (f < nf) {
        const uint32_t gf = a.flist[td.first + f];
        const cl_func fn = in.func[gf];
        const uint32_t b0 = in.func_blk_off[gf], b1 = in.func_blk_off[gf + 1];
        const uint32_t i0 = in.blk_off[b0], nrec = in.blk_off[b1] - i0;
        const uint32_t nimm = in.imm_off[gf + 1] - in.imm_off[gf];
        T.f_gf[f] = gf; T.f_gb0[f] = b0; T.f_gi0[f] = i0;
        T.f_arch[f] = fn.arch; T.f_nvid[f] = fn.next_vid; T.f_niid[f] = fn.next_iid; T.f_ntemp[f] = fn.next_temp_reg;
        T.f_nimm[f] = nimm; T.f_stat[f] = 0; T.f_nev[f] = 0; T.f_odd[f] = 0;
        T.f_mbase[f] = in.mem_off[gf]; T.f_nin[f] = nrec;
        T.f_oi[f] = tile_vcap(fn.next_vid, nrec); T.f_oq[f] = tile_qcap(nimm, nrec);     /* slice sizes, scanned below */
        T.f_ov[f] = b1 - b0;
        T.f_active[f] = 0; T.f_gate[f] = 0; T.f_rgate[f] = 0; T.f_chg[f] = 0; T.f_red[f] = 0; T.f_aux[f] = 0;
    }
    GFOR(g, k, nf * 64) if (k < nf * 64) (&T.f_stats[0][0])[k] = 0;
    g.sync();
    if (g.rank == 0) {
        uint32_t vb = 0, qb = 0, bb = 0, ib = 0;
        for (uint32_t f = 0; f < nf; f++) {
            T.f_vbase[f] = vb; T.f_qbase[f] = qb; T.f_b0[f] = bb; T.f_i0[f] = ib;
            vb += T.f_oi[f]; qb += T.f_oq[f]; bb += T.f_ov[f]; ib += T.f_nin[f];
        }
        T.f_vbase[nf] = vb; T.f_qbase[nf] = qb; T.f_b0[nf] = bb; T.f_i0[nf] = ib;
        T.vtot = vb; T.qtot = qb; T.nb = bb; T.n = ib;
        if (vb > C::V || qb > C::Q || ib > C::I || bb > C::B || nf > C::F) T.fail = 1;      /* planner bug: loud */
    }
    g.sync();
    if (T.fail) return;
    const uint32_t nb = T.nb, n = T.n;
    GFOR(g, b, nb) if (b < nb) {
        const uint32_t f = t_slice_of(T.f_b0, nf, b), gb = T.f_gb0[f] + (b - T.f_b0[f]);
        T.bfun[b] = (uint8_t)f;
        T.bo[b] = T.f_i0[f] + (in.blk_off[gb] - T.f_gi0[f]);
        cl_blk bk = in.blk[gb];
        for (int k = 0; k < 2; k++) if (kind_of(bk.term_tag[k]) == CL_K_VALUE) bk.term_pay[k] += T.f_vbase[f];
        T.blk[b] = bk;
    }
    if (g.rank == 0) T.bo[nb] = n;
    /* records: coalesced per function; value / immediate / memref ids rebased into the tile's index spaces */
    GFOR(g, i, n) if (i < n) {
        const uint32_t f = t_slice_of(T.f_i0, nf, i);
        const size_t src = (size_t)T.f_gi0[f] + (i - T.f_i0[f]);
        T.fidx[i] = (uint8_t)f;
        *(uint4 *)&T.hdr[i] = *(const uint4 *)(in.hdr + src);
        const uint4 tg4 = *(const uint4 *)(in.tag + src * 8);
        uint4 p0 = ((const uint4 *)(in.pay + src * 8))[0], p1 = ((const uint4 *)(in.pay + src * 8))[1];
        const uint16_t *tags = (const uint16_t *)&tg4;
        uint32_t *pp0 = (uint32_t *)&p0, *pp1 = (uint32_t *)&p1;
#pragma unroll
        for (unsigned k = 0; k < 4; k++) { pp0[k] = t_rebase(T, f, tags[k], pp0[k], true); pp1[k] = t_rebase(T, f, tags[4 + k], pp1[k], true); }
        *(uint4 *)&T.tag[(size_t)i * 8] = tg4;
        ((uint4 *)&T.pay[(size_t)i * 8])[0] = p0;
        ((uint4 *)&T.pay[(size_t)i * 8])[1] = p1;
    }
    for (uint32_t f = 0; f < nf; f++) {           /* memrefs: mutable copy in the output, value ids rebased */
        const uint32_t m0 = T.f_mbase[f], nm = in.mem_off[T.f_gf[f] + 1] - m0, vb = T.f_vbase[f];
        GFOR(g, m, nm) if (m < nm) {
            cl_memref r = in.mem[m0 + m];
            if (kind_of(r.base_tag) == CL_K_VALUE) r.base_pay += vb;
            if (kind_of(r.ureg_tag) == CL_K_VALUE) r.ureg_pay += vb;
            tg.mem[m0 + m] = r;
        }
    }
    GFOR(g, k, T.vtot) if (k < T.vtot) {
        const uint32_t f = t_slice_of(T.f_vbase, nf, k), v = k - T.f_vbase[f];
        const uint32_t v0 = in.val_off[T.f_gf[f]];
        const bool have = v < T.f_nvid[f];
        T.alive[k] = have ? in.val_alive[v0 + v] : (uint8_t)0;
        T.def_iid[k] = have ? in.val_def_iid[v0 + v] : -1;
        T.origin[k] = CL_ORG_HOST;
    }
    GFOR(g, k, T.qtot) if (k < T.qtot) {
        const uint32_t f = t_slice_of(T.f_qbase, nf, k), q = k - T.f_qbase[f];
        if (q < T.f_nimm[f]) T.imm[k] = in.imm[in.imm_off[T.f_gf[f]] + q];
    }
    g.sync();
    t_index(g, T);
}

/* results of the live functions go to one atomically reserved place per tile (function
 * order inside it); dead ones are queued for the general kernel                 */
template <class G, class C> CLF void t_store(const G &g, TileS<C> &T, const TileG<C> &tg, const TileIO &a) {
    PROF(g, T.fs, PF_STORE);
    const uint32_t nf = T.nf;
    /* tombstones leave here: live(x) = live records before position x */
    const uint32_t n_live = t_scan(g, T.n, [&](uint32_t p) { return (uint32_t)(T.hdr[p].op != CL_OP_TOMB); },
                                   [&](uint32_t p, uint32_t x) { T.outpos[p] = (uint16_t)x; });
    g.sync();
    auto live = [&](uint32_t x) -> uint32_t { return x < T.n ? (uint32_t)T.outpos[x] : n_live; };
    if (g.rank == 0) {
        uint32_t oi = 0, oq = 0, ov = 0, oe = 0;
        const bool tile_ok = !T.fail;
        for (uint32_t f = 0; f < nf; f++) {
            const bool ok = tile_ok && T.f_stat[f] == 0;
#if !CL_DEV
            if (!ok && getenv("CL_TILE_DEBUG")) fprintf(stderr, "tile hand-back: function %u (%u records) reason %u tile_fail %u\n", T.f_gf[f], T.f_nin[f], T.f_stat[f], T.fail);
#endif
            if (!ok && T.f_stat[f] == 0) T.f_stat[f] = CL_ST_REDO;
            T.f_oi[f] = oi; T.f_oq[f] = oq; T.f_ov[f] = ov; T.f_oe[f] = oe;
            if (ok) { oi += live(T.bo[T.f_b0[f + 1]]) - live(T.bo[T.f_b0[f]]); oq += T.f_nimm[f]; ov += T.f_nvid[f]; oe += T.f_nev[f]; }
        }
        const uint32_t ri = (uint32_t)a_add64(&a.cursor[0], oi), rq = (uint32_t)a_add64(&a.cursor[1], oq),
                       rv = (uint32_t)a_add64(&a.cursor[2], ov), re = (uint32_t)a_add64(&a.cursor[3], oe);
        const bool fits = (unsigned long long)ri + oi <= a.cap[0] && (unsigned long long)rq + oq <= a.cap[1] &&
                          (unsigned long long)rv + ov <= a.cap[2] && (unsigned long long)re + oe <= a.cap[3];
        unsigned long long n_in = 0;
        for (uint32_t f = 0; f < nf; f++) {
            T.f_oi[f] += ri; T.f_oq[f] += rq; T.f_ov[f] += rv; T.f_oe[f] += re;
            T.f_aux[f] = 0;
            if (T.f_stat[f] == 0) n_in += T.f_nin[f];
        }
        T.work = fits ? 1u : 0u;
        a_add64(&a.stats[64], n_in); a_add64(&a.stats[65], oi); a_add64(&a.stats[66], oe);
    }
    g.sync();
    const bool fits = T.work != 0;
    TFuncOut *o_func = (TFuncOut *)a.o_func;
    GFOR(g, f, nf) if (f < nf) {
        if (T.f_stat[f] != 0) {
#if !CL_DEV
            if (getenv("CL_DEBUG_REDO")) fprintf(stderr, "tile hand-back: function %u (%u records) status %u\n", T.f_gf[f], T.f_nin[f], T.f_stat[f]);
#endif
            if (T.f_nin[f] > a.small_max) a.retry_big_list[a_add(a.retry_big_count, 1u)] = T.f_gf[f];
            else a.retry_list[a_add(a.retry_count, 1u)] = T.f_gf[f];
            continue;
        }
        const uint32_t cnt = live(T.bo[T.f_b0[f + 1]]) - live(T.bo[T.f_b0[f]]);
        TFuncOut o;
        o.f.next_vid = T.f_nvid[f]; o.f.next_iid = T.f_niid[f]; o.f.next_temp_reg = T.f_ntemp[f];
        o.f.arch = T.f_arch[f]; o.f.status = (uint8_t)(fits ? CL_ST_OK : CL_ST_CAPACITY); o.f.reserved = 0;
        o.inst_start = T.f_oi[f]; o.n_inst = fits ? cnt : 0; o.imm_start = T.f_oq[f]; o.n_imm = fits ? T.f_nimm[f] : 0;
        o.val_start = T.f_ov[f]; o.ev_start = T.f_oe[f]; o.n_ev = fits ? T.f_nev[f] : 0; o.pad = 0;
        o_func[T.f_gf[f]] = o;
    }
    GFOR(g, b, T.nb) if (b < T.nb) {
        const uint32_t f = T.bfun[b];
        if (T.f_stat[f] != 0) continue;
        cl_blk bk = T.blk[b];
        for (int k = 0; k < 2; k++) bk.term_pay[k] = t_rebase(T, f, bk.term_tag[k], bk.term_pay[k], false);
        const uint32_t gb = T.f_gb0[f] + (b - T.f_b0[f]);
        a.o_blk[gb] = bk;
        a.o_blk_start[gb] = fits ? T.f_oi[f] + (live(T.bo[b]) - live(T.bo[T.f_b0[f]])) : 0u;
        a.o_blk_cnt[gb] = fits ? live(T.bo[b + 1]) - live(T.bo[b]) : 0u;
    }
    /* memrefs of the live functions back to function-local value ids (dead ones are reloaded by the general kernel) */
    for (uint32_t f = 0; f < nf; f++) {
        if (T.f_stat[f] != 0) continue;
        const uint32_t m0 = T.f_mbase[f], nm = a.in.mem_off[T.f_gf[f] + 1] - m0, vb = T.f_vbase[f];
        GFOR(g, m, nm) if (m < nm) {
            cl_memref &r = tg.mem[m0 + m];
            if (kind_of(r.base_tag) == CL_K_VALUE) r.base_pay -= vb;
            if (kind_of(r.ureg_tag) == CL_K_VALUE) r.ureg_pay -= vb;
        }
    }
    if (fits) {
        GFOR(g, i, T.n) if (i < T.n) {
            const uint32_t f = T.fidx[i];
            if (T.f_stat[f] != 0 || T.hdr[i].op == CL_OP_TOMB) continue;
            const size_t d = (size_t)T.f_oi[f] + (live(i) - live(T.bo[T.f_b0[f]]));
            uint4 tg4 = *(const uint4 *)&T.tag[(size_t)i * 8];
            uint4 p0 = ((const uint4 *)&T.pay[(size_t)i * 8])[0], p1 = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
            const uint16_t *tags = (const uint16_t *)&tg4;
            uint32_t *pp0 = (uint32_t *)&p0, *pp1 = (uint32_t *)&p1;
#pragma unroll
            for (unsigned k = 0; k < 4; k++) { pp0[k] = t_rebase(T, f, tags[k], pp0[k], false); pp1[k] = t_rebase(T, f, tags[4 + k], pp1[k], false); }
            *(uint4 *)(a.o_hdr + d) = *(const uint4 *)&T.hdr[i];
            *(uint4 *)(a.o_tag + d * 8) = tg4;
            ((uint4 *)(a.o_pay + d * 8))[0] = p0;
            ((uint4 *)(a.o_pay + d * 8))[1] = p1;
        }
        GFOR(g, k, T.qtot) if (k < T.qtot) {
            const uint32_t f = t_slice_of(T.f_qbase, nf, k), q = k - T.f_qbase[f];
            if (T.f_stat[f] == 0 && q < T.f_nimm[f]) a.o_imm[T.f_oq[f] + q] = T.imm[k];
        }
        GFOR(g, k, T.vtot) if (k < T.vtot) {
            const uint32_t f = t_slice_of(T.f_vbase, nf, k), v = k - T.f_vbase[f];
            if (T.f_stat[f] == 0 && v < T.f_nvid[f]) {
                const size_t d = (size_t)T.f_ov[f] + v;
                a.o_alive[d] = T.alive[k]; a.o_def_iid[d] = T.def_iid[k]; a.o_origin[d] = T.origin[k];
            }
        }
        const uint32_t nev = T.n_ev < C::E ? T.n_ev : C::E;
        GFOR(g, e, nev) if (e < nev) {
            cl_event ev = tg.ev[e];
            const uint32_t f = ev.func;
            ev.func = T.f_gf[f];
            if (T.f_stat[f] == 0) a.o_ev[T.f_oe[f] + a_add(&T.f_aux[f], 1u)] = ev;
        }
    }
    GFOR(g, k, 64) if (k < 64) {
        unsigned long long sum = 0;
        for (uint32_t f = 0; f < nf; f++) if (T.f_stat[f] == 0) sum += T.f_stats[f][k];
        if (sum) a_add64(&a.stats[k], sum);
    }
    g.sync();
}

/* the four calls of pipeline.py:165-169 on every function of one tile         */
template <class G, class C> CLF void t_set_gate(const G &g, TileS<C> &T, int mode) {
    /* 0: live sm52 functions, 1: live active functions, 2: live functions with redirects, 3: all live */
    GFOR(g, f, T.nf) if (f < T.nf) {
        bool on = tf_ok(T, f);
        if (mode == 0) on = on && T.f_arch[f] == CL_ARCH_SM52;
        else if (mode == 1) on = on && T.f_active[f];
        else if (mode == 2) on = on && T.f_red[f] != 0;
        T.f_gate[f] = on;
    }
    g.sync();
}
template <class G, class C> CLD bool t_any_gate(const G &g, TileS<C> &T) {
    bool m = false;
    GFOR(g, f, T.nf) if (f < T.nf) m |= T.f_gate[f] != 0;
    return g.any(m);
}

template <class G, class C> CLF void t_run_tile(const G &g, TileS<C> &T, TileG<C> &tg, const TileIO &a, const TileDesc td) {
    const uint32_t passes = T.fs.passes, max_rounds = T.fs.max_rounds;
    t_load(g, T, tg, a, td);
    if (!T.fail && (passes & CL_PASS_XMAD)) {
        t_set_gate(g, T, 0);
        if (t_any_gate(g, T)) {
            t_apply_patterns(g, T, tg, 1, 0);
            if (!T.fail) t_dce(g, T, tg);
        }
    }
    if (!T.fail && (passes & CL_PASS_RECIPROCAL)) t_reciprocal(g, T, tg);
    if (!T.fail && (passes & CL_PASS_AGGREGATE)) {
        GFOR(g, f, T.nf) if (f < T.nf) T.f_active[f] = 1;
        g.sync();
        for (uint32_t round = 0; round < max_rounds && !T.fail; round++) {
            t_set_gate(g, T, 1);
            if (!t_any_gate(g, T)) break;
            GFOR(g, f, T.nf) if (f < T.nf) T.f_chg[f] = 0;
            g.sync();
            t_apply_patterns(g, T, tg, 0, 2 + round);
            if (T.fail) break;
            t_set_gate(g, T, 1);
            t_simplify(g, T, tg);
            t_set_gate(g, T, 2);
            if (t_any_gate(g, T)) t_dce(g, T, tg);
            GFOR(g, f, T.nf) if (f < T.nf) T.f_active[f] = T.f_active[f] && (T.f_chg[f] + T.f_red[f]) != 0;
            g.sync();
        }
        if (!T.fail) { t_set_gate(g, T, 3); t_dce(g, T, tg); }
    }
    if (!T.fail && (passes & CL_PASS_TAG)) t_tag(g, T);
    g.sync();
    t_store(g, T, tg, a);
}

/* once per CTA: the pattern table in shared memory, seed classes of both tables,
 * anchors, unification constraints.  `fs` is any FS whose pb can be pointed at P. */
template <class G> CLF void t_setup(const G &g, TileP &P, const cl_pattern_blob *pb) {
    {
        const uint32_t *src = (const uint32_t *)pb;
        uint32_t *dst = (uint32_t *)&P.pb;
        GFOR(g, k, sizeof(cl_pattern_blob) / 4) if (k < sizeof(cl_pattern_blob) / 4) dst[k] = src[k];
        GFOR(g, k, 2 * CL_OP__COUNT) if (k < 2 * CL_OP__COUNT) (&P.op_cls[0][0])[k] = 0xFF;
    }
    g.sync();
    if (g.rank == 0) {
        for (unsigned table = 0; table < 2; table++) {
            unsigned n_cls = 0;
            for (unsigned c = 0; c < (unsigned)MAX_CLS; c++) { P.cls_op[table][c] = 0xFFFF; P.anchor_mask[table][c] = 0; }
            for (unsigned pi = 0; pi < P.pb.n_patterns; pi++) {
                const cl_pattern &p = P.pb.p[pi];
                if (p.table != table) continue;
                for (unsigned t = 0; t < p.n_templates; t++) {
                    bool seen = false;
                    for (unsigned c = 0; c < n_cls; c++) seen |= P.cls_op[table][c] == p.t[t].op;
                    if (!seen && n_cls < (unsigned)MAX_CLS) P.cls_op[table][n_cls++] = p.t[t].op;
                }
            }
            P.n_cls[table] = n_cls;
            for (unsigned c = 0; c < n_cls; c++) if (P.cls_op[table][c] < CL_OP__COUNT) P.op_cls[table][P.cls_op[table][c]] = (uint8_t)c;
            for (unsigned pi = 0; pi < P.pb.n_patterns; pi++) {
                const cl_pattern &p = P.pb.p[pi];
                if (p.table != table) continue;
                const uint16_t aop = p.t[p.join_order[0]].op;
                for (unsigned c = 0; c < n_cls; c++) if (P.cls_op[table][c] == aop) P.anchor_mask[table][c] |= 1u << pi;
            }
        }
    }
    GFOR(g, pi, P.pb.n_patterns) if (pi < P.pb.n_patterns) {
        const cl_pattern &p = P.pb.p[pi];
        TPat &tp = P.pat[pi];
        tp.n_pairs = tp.n_mpairs = 0;
        uint8_t ft[CL_MAX_VARS], fk[CL_MAX_VARS], mt[CL_MAX_GROUPS], mg[CL_MAX_GROUPS];
        for (int v = 0; v < CL_MAX_VARS; v++) ft[v] = 0xFF;
        for (int v = 0; v < CL_MAX_GROUPS; v++) mt[v] = 0xFF;
        for (unsigned t = 0; t < p.n_templates; t++) {
            const cl_template &tm = p.t[t];
            for (unsigned k = 0; k < tm.n_modvars; k++) {
                const unsigned mv = tm.modvar_var[k] & (CL_MAX_GROUPS - 1);
                if (mt[mv] == 0xFF) { mt[mv] = (uint8_t)t; mg[mv] = tm.modvar_group[k]; }
                else if (tp.n_mpairs < 4) { uint8_t *m = tp.mpair[tp.n_mpairs++]; m[0] = mt[mv]; m[1] = mg[mv]; m[2] = (uint8_t)t; m[3] = tm.modvar_group[k]; }
            }
            const unsigned ns = (unsigned)tm.n_defs + tm.n_aux + tm.n_uses;
            for (unsigned k = 0; k < ns && k < 8; k++) {
                if (tm.slot[k].kind != CL_S_VAR) continue;
                const unsigned v = tm.slot[k].var & (CL_MAX_VARS - 1);
                if (ft[v] == 0xFF) { ft[v] = (uint8_t)t; fk[v] = (uint8_t)k; }
                else if (tp.n_pairs < 28) { uint8_t *m = tp.pair[tp.n_pairs++]; m[0] = ft[v]; m[1] = fk[v]; m[2] = (uint8_t)t; m[3] = (uint8_t)k; }
            }
        }
    }
    g.sync();
}

} /* namespace clk */

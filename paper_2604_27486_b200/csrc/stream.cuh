/* stream.cuh -- the post-SSA stage as corpus-wide streaming passes.
 *
 * tile.cuh showed that the stage can be evaluated for many functions at once
 * on the def-use snapshot of a pass (one thread per record / candidate /
 * selected match, hazards detected and handed back).  Its tiles are small, so
 * every CTA walks ~300 KB of code for a few thousand records and waits on
 * L2 latency with a handful of warps.  Here the "tile" is the whole corpus:
 * all functions live in corpus-wide index spaces in HBM, the group is the
 * whole (cooperatively launched) grid, and every pass is one coalesced sweep
 * over a plane of the stream -- the seed scan, unification, selection and
 * rewrite passes of the north star, separated by grid barriers:
 *
 *   s_load       rebase ids into corpus-wide spaces        (64 B/record in, 72 out)
 *   s_usecount   def positions + use counts (L2 atomics)   ssa.py:613-636
 *   s_match      seed classes -> (anchor, pattern) work list by prefix sum ->
 *                join unification per item                 patterns.py:130-216
 *   s_select     atomicMin bidding fixpoint over the raw matches  :241-252
 *   s_apply      plan one selected match per thread, id bases by prefix sums,
 *                stream permutation into the second buffer :671-707
 *   s_simplify / s_dce / s_reciprocal / s_tag              :710-916
 *   s_store      ids back to function-local, dense result in function order
 *
 * Exactness is tile.cuh's argument unchanged: functions are independent, every
 * pass sees the snapshot of its start, sequential hazards (G5 cross-block
 * escapes, interfering reciprocal chains, RZ/PT join links, reference
 * exceptions, slice overflow) mark the function and it is redone by the
 * general per-function kernel of core.cuh.
 */
#pragma once
#include "core.cuh"
#include "kargs.h"
#if CL_DEV
#include <cooperative_groups.h>
#endif

namespace clk {

static constexpr uint32_t CLS_REDO = 100;       /* internal status: redo this function on the general kernel */
static constexpr uint32_t CLS_BIG_BLOCK = 37;   /* below this many records no candidate product reaches the 50 000 budget (36^3) */

struct SMatch { uint32_t pos[3]; uint8_t pat, n; uint16_t pad; };
struct SChain { uint32_t add, mufu, rcp, addv, f, rank; };
struct SPat {
    uint8_t n_pairs, n_mpairs, pad[2];
    uint8_t pair[28][4];       /* tA, kA, tB, kB: slots in defs, aux, uses order    */
    uint8_t mpair[4][4];       /* tA, groupA, tB, groupB                            */
};
/* the pattern table and what s_setup derives from it (one copy in global memory) */
struct StreamP {
    cl_pattern_blob pb;
    SPat pat[CL_MAX_PATTERNS];
    uint16_t cls_op[2][MAX_CLS];
    uint32_t n_cls[2], anchor_mask[2][MAX_CLS];
    uint8_t op_cls[2][CL_OP__COUNT];      /* opcode id -> seed class of the table, 0xFF none */
};

struct StreamCaps { uint32_t I, V, Q, M, S, X, E; };
enum { SP_LOAD = 0, SP_USECOUNT, SP_SEED, SP_ITEMS, SP_BUDGET, SP_UNIFY, SP_SELECT, SP_SELSCAN, SP_PLAN, SP_BASES, SP_MARK, SP_PERMUTE,
       SP_STAGE, SP_SIMPLIFY, SP_DCE, SP_RECIP, SP_TAG, SP_STORE, SP_GATE, SP__N = 24 };

/* everything the passes touch; lives in global memory, arrays sized by the host (stream.cu) */
struct StreamS {
    /* the stream: live buffer and the one the next permutation writes */
    cl_hdr *hdr, *hdr2; uint16_t *tag, *tag2; uint32_t *pay, *pay2;
    uint32_t *fidx, *fidx2, *bidx, *bidx2;
    unsigned long long *owner;                                   /* [I] */
    uint32_t *outpos, *sel_at;                                   /* [I] */
    uint8_t *keep, *inscnt, *clsid, *flag;                       /* [I] */
    uint32_t *usecnt, *defpos, *redirect, *origin; int32_t *def_iid; uint8_t *alive;      /* [V] */
    cl_imm *imm;                                                 /* [Q] */
    SelRec *sel; Stage *stage;                                   /* [S] */
    SMatch *mt; uint8_t *mstate;                                 /* [M] */
    SChain *chain;                                               /* [X] */
    cl_event *ev;                                                /* [E] */
    cl_memref *mem;                                              /* mutable copy in the output */
    /* blocks */
    uint32_t *bo, *bo2, *b_first, *bfun; cl_blk *blk;            /* [B + 1] / [B]; blk = mutable copy in the output */
    uint32_t (*ccnt)[MAX_CLS]; uint32_t (*cbase)[MAX_CLS]; uint16_t *b_over;
    /* functions */
    uint32_t *f_vbase, *f_qbase;                                 /* [F + 1] slices of the value / immediate spaces */
    const uint32_t *f_b0, *f_mbase;                              /* [F + 1] first block / first memref (the input's CSR offsets) */
    uint32_t *f_nvid, *f_niid, *f_nimm, *f_stat, *f_nev, *f_chg, *f_red, *f_first, *f_aux, *f_nin;
    uint32_t *f_oi, *f_oq, *f_ov, *f_oe;
    uint32_t (*f_stats)[64];
    uint8_t *f_arch, *f_active, *f_odd, *f_gate;
    const StreamP *P;
    FS fs;
    StreamCaps cap;
    uint32_t n, nb, nf, n_mt, n_sel, n_ev, fail, vtot, qtot, n_chain, n_items, work;
    uint32_t res[4];                                             /* places reserved in the result buffers */
    uint32_t du_ok;                                              /* usecnt / defpos describe the stream for the gated functions */
    unsigned long long prof[SP__N], prof_t0;                     /* nanoseconds per phase (lane 0 of the grid) */
    uint32_t iters[4];                                           /* select / dce fixpoint iterations, rounds */
    uint32_t rstat[8][4];                                        /* per apply_patterns call: gated records, work items, raw matches, selected */
    uint32_t n_apply;
    uint32_t redo[24];                                           /* hand-backs by reason (status - CLS_REDO), [23]: whole-stage failure */
};

struct StreamIO {              /* the part of KArgs the stream kernel needs */
    cl_corpus in;
    cl_hdr *o_hdr; uint16_t *o_tag; uint32_t *o_pay; cl_imm *o_imm;
    uint8_t *o_alive; int32_t *o_def_iid; uint32_t *o_origin;
    cl_memref *o_mem;
    cl_blk *o_blk; uint32_t *o_blk_start, *o_blk_cnt;
    cl_event *o_ev;
    FuncOut *o_func;
    unsigned long long cap[4];
    unsigned long long *cursor, *stats;
    uint32_t *retry_list, *retry_count;
    uint32_t *retry_big_list, *retry_big_count; uint32_t small_max;
    uint32_t passes, max_rounds;
};

/* ------------------------------------------------------------------ the group */
#if CL_DEV
/* the whole grid as one group (cooperative launch: every CTA is resident)       */
struct GridGrp {
    uint32_t rank, size;
    uint32_t *part;            /* [gridDim.x] scan partials (global)                */
    uint32_t *slots;           /* [3] rotating reduction words (global, zero at launch) */
    Grp<8> cta;                /* 256 threads                                       */
    mutable uint32_t turn;
    CLD void sync() const { cooperative_groups::this_grid().sync(); }
    CLD uint32_t *turn_slot() const {
        uint32_t *s = slots + turn % 3u;
        if (rank == 0) slots[(turn + 1u) % 3u] = 0;       /* nobody reads or writes it during this turn */
        turn++;
        return s;
    }
    CLD bool any(bool f) const {
        const int c = __syncthreads_or(f);
        uint32_t *s = turn_slot();
        if (threadIdx.x == 0 && c) atomicOr(s, 1u);
        sync();
        return *(volatile uint32_t *)s != 0;
    }
    CLD uint32_t any_bits(uint32_t x) const {           /* bitwise or over the grid */
        const uint32_t w = __reduce_or_sync(0xFFFFFFFFu, x);
        uint32_t *s = turn_slot();
        if ((threadIdx.x & 31u) == 0 && w) atomicOr(s, w);
        sync();
        return *(volatile uint32_t *)s;
    }
    CLD uint32_t sum(uint32_t x) const {
        const uint32_t c = cta.sum(x);
        uint32_t *s = turn_slot();
        if (threadIdx.x == 0 && c) atomicAdd(s, c);
        sync();
        return *(volatile uint32_t *)s;
    }
    CLD uint32_t wrank() const { return rank >> 5; }
    CLD uint32_t wcount() const { return size >> 5; }
    CLD uint32_t lane() const { return rank & 31u; }
    CLD uint32_t lanes() const { return 32u; }
};
/* one address, many lanes: one atomic per warp */
CLD uint32_t a_inc_agg(uint32_t *p) {
    const uint32_t mask = __activemask(), lane = threadIdx.x & 31u;
    const int leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if ((int)lane == leader) base = atomicAdd(p, (uint32_t)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(mask & ((1u << lane) - 1u));
}
/* exclusive scan over items [0, n) in order, grid wide: every CTA owns a contiguous run of items,
 * sums it, waits for the others, rescans it from its base.  `in` is evaluated twice per item.     */
template <class FIN, class FOUT> CLD uint32_t s_scan(const GridGrp &g, uint32_t n, FIN in, FOUT out) {
    constexpr uint32_t K = 8;                                   /* consecutive items per thread and step: K loads in flight */
    const uint32_t nc = gridDim.x, bt = blockDim.x, c = blockIdx.x, t = threadIdx.x, step = bt * K;
    uint32_t L = (n + nc - 1) / nc;
    L = (L + step - 1) / step * step;
    const unsigned long long lo64 = (unsigned long long)c * L;
    const uint32_t lo = lo64 < n ? (uint32_t)lo64 : n, hi = n - lo < L ? n : lo + L;
    uint32_t s = 0;
    for (uint32_t j0 = lo + t * K; j0 < hi; j0 += step) {
        uint32_t x[K];
#pragma unroll
        for (uint32_t k = 0; k < K; k++) x[k] = j0 + k < hi ? in(j0 + k) : 0u;
#pragma unroll
        for (uint32_t k = 0; k < K; k++) s += x[k];
    }
    const uint32_t tot = g.cta.sum(s);
    if (t == 0) g.part[c] = tot;
    g.sync();
    uint32_t before = 0, all = 0;
    for (uint32_t k = t; k < nc; k += bt) { const uint32_t p = *(volatile uint32_t *)&g.part[k]; all += p; if (k < c) before += p; }
    before = g.cta.sum(before);
    all = g.cta.sum(all);
    uint32_t run = before;
    for (uint32_t base = lo; base < hi; base += step) {
        const uint32_t j0 = base + t * K;
        uint32_t x[K], mine = 0;
#pragma unroll
        for (uint32_t k = 0; k < K; k++) { x[k] = j0 + k < hi ? in(j0 + k) : 0u; }
#pragma unroll
        for (uint32_t k = 0; k < K; k++) mine += x[k];
        uint32_t tt;
        uint32_t o = run + g.cta.exscan(mine, tt);
#pragma unroll
        for (uint32_t k = 0; k < K; k++) { if (j0 + k < hi) out(j0 + k, o); o += x[k]; }
        run += tt;
    }
    g.sync();
    return all;
}
#endif
/* the one-lane host group (tests/sim): same code, collectives are identities    */
CLD uint32_t g_wrank(const Grp<0> &) { return 0; }
CLD uint32_t g_wcount(const Grp<0> &) { return 1; }
CLD uint32_t g_lane(const Grp<0> &) { return 0; }
CLD uint32_t g_lanes(const Grp<0> &) { return 1; }
CLD uint32_t g_any_bits(const Grp<0> &, uint32_t x) { return x; }
#if CL_DEV
CLD uint32_t g_any_bits(const GridGrp &g, uint32_t x) { return g.any_bits(x); }
CLD uint32_t g_wrank(const GridGrp &g) { return g.wrank(); }
CLD uint32_t g_wcount(const GridGrp &g) { return g.wcount(); }
CLD uint32_t g_lane(const GridGrp &g) { return g.lane(); }
CLD uint32_t g_lanes(const GridGrp &g) { return g.lanes(); }
#else
CLD uint32_t a_inc_agg(uint32_t *p) { return a_add(p, 1u); }
#endif
template <class FIN, class FOUT> CLD uint32_t s_scan(const Grp<0> &, uint32_t n, FIN in, FOUT out) {
    uint32_t run = 0;
    for (uint32_t j = 0; j < n; j++) { const uint32_t x = in(j); (void)in(j); out(j, run); run += x; }
    return run;
}
/* independent strided loop (no collectives inside)                             */
#define SFOR(g, i, n) for (uint32_t i = (g).rank; i < (n); i += (g).size)
/* one warp per item f, lanes over its parts                                     */
#define WFOR(g, f, n) for (uint32_t f = g_wrank(g); f < (n); f += g_wcount(g))
#define LFOR(g, k, n) for (uint32_t k = g_lane(g); k < (n); k += g_lanes(g))

/* phase clock: lane 0 of the grid charges the time since the previous mark to `slot` */
template <class G> CLD void s_mark(const G &g, StreamS &T, int slot) {
#if CL_DEV
    if (g.rank == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        T.prof[slot] += t - T.prof_t0;
        T.prof_t0 = t;
    }
#else
    (void)g; (void)T; (void)slot;
#endif
}
CLD bool sf_ok(const StreamS &T, uint32_t f) { return *(volatile const uint32_t *)&T.f_stat[f] == 0; }
/* a failed function leaves the gate at once, so sweeps that look at the gate need no second look-up */
CLD void sf_fail(StreamS &T, uint32_t f, uint32_t code) { a_cas0(&T.f_stat[f], code); *(volatile uint8_t *)&T.f_gate[f] = 0; }
CLD bool sf_on(const StreamS &T, uint32_t f) { return *(volatile const uint8_t *)&T.f_gate[f] != 0; }
CLD void s_fail(StreamS &T) { *(volatile uint32_t *)&T.fail = 1; }

CLD void s_event(StreamS &T, uint32_t f, uint32_t seq, uint32_t kind, uint32_t idx, uint32_t a, uint32_t b) {
    const uint32_t k = a_inc_agg(&T.n_ev);
    if (k < T.cap.E) {
        cl_event e; e.func = f; e.seq = seq; e.kind = kind; e.idx = idx; e.a = a; e.b = b; e.c = 0; e.d = 0;
        T.ev[k] = e;
        a_add(&T.f_nev[f], 1u);
    } else
        s_fail(T);
}
CLD int s_class_of(const StreamS &T, unsigned table, uint16_t op) {
    if (op >= CL_OP__COUNT) return -1;            /* dynamic opcodes never head a template */
    const uint8_t c = T.P->op_cls[table][op];
    return c == 0xFF ? -1 : (int)c;
}
CLD opnd s_slot(const StreamS &T, uint32_t i, unsigned k) {
    opnd o; o.tag = T.tag[(size_t)i * 8 + k]; o.pay = T.pay[(size_t)i * 8 + k];
    return o;
}
/* one record in registers: passes that look at most slots load it with four 128-bit loads */
struct RecR { cl_hdr h; uint16_t tag[8]; uint32_t pay[8]; };
CLD RecR s_rec(const StreamS &T, uint32_t i) {
    RecR r;
    *(uint4 *)&r.h = *(const uint4 *)&T.hdr[i];
    *(uint4 *)r.tag = *(const uint4 *)&T.tag[(size_t)i * 8];
    ((uint4 *)r.pay)[0] = ((const uint4 *)&T.pay[(size_t)i * 8])[0];
    ((uint4 *)r.pay)[1] = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
    return r;
}
/* value_operands (ssa.py:599-610) / all_defs of a record without overflow slots */
template <class F> CLD void s_value_operands(const StreamS &T, const cl_hdr &h, uint32_t i, F fn) {
    if (has_guard(h)) { const opnd g = s_slot(T, i, 0); if (is_value(g)) fn(g.pay); }
    const unsigned u0 = use0(h);
    for (unsigned k = 0; k < h.n_uses; k++) {
        const opnd u = s_slot(T, i, u0 + k);
        if (is_value(u)) fn(u.pay);
        else if (kind_of(u.tag) == CL_K_MEMREF) {
            const cl_memref &m = T.mem[u.pay];
            if (kind_of(m.base_tag) == CL_K_VALUE) fn(m.base_pay);
            if (kind_of(m.ureg_tag) == CL_K_VALUE) fn(m.ureg_pay);
        }
    }
}
template <class F> CLD void s_value_defs(const StreamS &T, const cl_hdr &h, uint32_t i, F fn) {
    const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
    for (unsigned k = 0; k < nd; k++) { const opnd d = s_slot(T, i, d0 + k); if (is_value(d)) fn(d.pay); }
}
/* the same on a record held in registers                                       */
template <class F> CLD void r_value_operands(const StreamS &T, const RecR &r, F fn) {
    const cl_hdr &h = r.h;
    if (has_guard(h) && kind_of(r.tag[0]) == CL_K_VALUE) fn(r.pay[0]);
    const unsigned u0 = use0(h);
#pragma unroll
    for (unsigned k = 0; k < 8; k++) {
        if (k < u0 || k >= u0 + h.n_uses) continue;
        const unsigned kd = kind_of(r.tag[k]);
        if (kd == CL_K_VALUE) fn(r.pay[k]);
        else if (kd == CL_K_MEMREF) {
            const cl_memref &m = T.mem[r.pay[k]];
            if (kind_of(m.base_tag) == CL_K_VALUE) fn(m.base_pay);
            if (kind_of(m.ureg_tag) == CL_K_VALUE) fn(m.ureg_pay);
        }
    }
}
template <class F> CLD void r_value_defs(const RecR &r, F fn) {
    const unsigned d0 = def0(r.h), nd = (unsigned)r.h.n_defs + r.h.n_aux;
#pragma unroll
    for (unsigned k = 0; k < 8; k++) if (k >= d0 && k < d0 + nd && kind_of(r.tag[k]) == CL_K_VALUE) fn(r.pay[k]);
}

/* permutation of the stream into the second buffer: record i moves to dst(i)
 * (NONE32 = dropped) with its function / block index; then the buffers swap.  */
template <class G, class F> CLD void s_permute(const G &g, StreamS &T, uint32_t n, F dst) {
    SFOR(g, i, n) {
        const uint32_t d = dst(i);
        if (d == NONE32) continue;
        const uint4 a = *(const uint4 *)&T.hdr[i], b = *(const uint4 *)&T.tag[(size_t)i * 8];
        const uint4 c0 = ((const uint4 *)&T.pay[(size_t)i * 8])[0], c1 = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
        const uint32_t f = T.fidx[i], bi = T.bidx[i];
        *(uint4 *)&T.hdr2[d] = a;
        *(uint4 *)&T.tag2[(size_t)d * 8] = b;
        ((uint4 *)&T.pay2[(size_t)d * 8])[0] = c0;
        ((uint4 *)&T.pay2[(size_t)d * 8])[1] = c1;
        T.fidx2[d] = f; T.bidx2[d] = bi;
    }
    g.sync();
    if (g.rank == 0) {
        cl_hdr *h = T.hdr; T.hdr = T.hdr2; T.hdr2 = h;
        uint16_t *t = T.tag; T.tag = T.tag2; T.tag2 = t;
        uint32_t *p = T.pay; T.pay = T.pay2; T.pay2 = p;
        uint32_t *x = T.fidx; T.fidx = T.fidx2; T.fidx2 = x;
        x = T.bidx; T.bidx = T.bidx2; T.bidx2 = x;
        T.fs.S.hdr = T.hdr; T.fs.S.tag = T.tag; T.fs.S.pay = T.pay;
    }
    g.sync();
}

/* new block offsets after a permutation described by outpos[] (position of the
 * first output slot of every old record) and the new length                   */
template <class G> CLD void s_rebase_blocks(const G &g, StreamS &T, uint32_t n_old, uint32_t n_new) {
    const uint32_t nb = T.nb;
    SFOR(g, b, nb + 1) { const uint32_t old = T.bo[b]; T.bo2[b] = old < n_old ? T.outpos[old] : n_new; }
    g.sync();
    if (g.rank == 0) { uint32_t *x = T.bo; T.bo = T.bo2; T.bo2 = x; T.n = n_new; T.fs.bo = T.bo; T.du_ok = 0; }
    g.sync();
    /* function-relative positions are compared as 16-bit numbers (s_key, chain order) */
    const uint32_t nf = T.nf;
    SFOR(g, f, nf) if (T.bo[T.f_b0[f + 1]] - T.bo[T.f_b0[f]] > 0xFFFFu) sf_fail(T, f, CLS_REDO + 14);
    g.sync();
}

/* ------------------------------------------------------------------ def-use */
/* ssa.py:613-636 for every gated live function at once (the others' words keep what they held) */
template <class G> CLF void s_usecount(const G &g, StreamS &T) {
    const uint32_t n = T.n, nb = T.nb, nf = T.nf, V = T.cap.V;
    WFOR(g, f, nf) {
        if (!sf_on(T, f)) continue;
        const uint32_t vb = T.f_vbase[f], room = T.f_vbase[f + 1] - vb;
        LFOR(g, v, room) { T.usecnt[vb + v] = 0; T.defpos[vb + v] = NONE32; }
    }
    g.sync();
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f)) continue;
        const RecR r = s_rec(T, i);
        const unsigned d0 = def0(r.h), nd = (unsigned)r.h.n_defs + r.h.n_aux;
        bool odd = false;
#pragma unroll
        for (unsigned k = 0; k < 8; k++) {
            if (k < d0 || k >= d0 + nd) continue;
            const unsigned kd = kind_of(r.tag[k]);
            if (kd == CL_K_VALUE) { if (r.pay[k] < V) T.defpos[r.pay[k]] = i; }
            else odd |= !(kd == CL_K_RZ || kd == CL_K_URZ || kd == CL_K_PRED);
        }
        if (odd) T.f_odd[f] = 1;
        r_value_operands(T, r, [&](uint32_t v) { if (v < V) a_add(&T.usecnt[v], 1u); });
    }
    SFOR(g, b, nb) {
        const uint32_t f = T.bfun[b];
        if (!sf_on(T, f)) continue;
        for (int k = 0; k < 2; k++)
            if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE && T.blk[b].term_pay[k] < V)
                a_add(&T.usecnt[T.blk[b].term_pay[k]], 1u);
    }
    if (g.rank == 0) T.du_ok = 1;
    g.sync();
    s_mark(g, T, SP_USECOUNT);
}

/* ----------------------------------------------------------------- matching */
/* operand_key equality (patterns.py:109-127) of two operands                   */
CLN bool s_key_equal(const StreamS &T, opnd a, opnd b) {
    unsigned ka = kind_of(a.tag), kb = kind_of(b.tag);
    if (ka == CL_K_URZ) ka = CL_K_RZ;
    if (kb == CL_K_URZ) kb = CL_K_RZ;
    const bool oa = ka == CL_K_NONE || ka >= CL_K_MEMREF, ob = kb == CL_K_NONE || kb >= CL_K_MEMREF;
    if (oa || ob) {
        if (!(oa && ob)) return false;
        const cl_memref &x = T.mem[a.pay], &y = T.mem[b.pay];       /* ("other", str(op)) */
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
CLN bool s_match_local(const StreamS &T, const cl_template &t, const cl_hdr &h, uint32_t i) {
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
        const opnd o = s_slot(T, i, g0 + k);
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
/* do two records share a value (defs and value operands of both)?  One edge of
 * _connected (patterns.py:219-238)                                            */
CLN bool s_linked(const StreamS &T, uint32_t i, uint32_t j) {
    /* kept small and out of line: inlined with its nested loops it made the unify loop 244 KB of code */
    const cl_hdr hi = T.hdr[i], hj = T.hdr[j];
    uint32_t a[16];                       /* <= 8 slots, a MemRef slot carries two values */
    unsigned na = 0;
    auto push = [&](uint32_t v) { if (na < 16) a[na++] = v; };
    s_value_defs(T, hi, i, push);
    s_value_operands(T, hi, i, push);
    bool hit = false;
    auto probe = [&](uint32_t w) { for (unsigned k = 0; k < na; k++) hit |= a[k] == w; };
    s_value_defs(T, hj, j, probe);
    s_value_operands(T, hj, j, probe);
    return hit;
}
/* one candidate tuple of match_patterns (patterns.py:199-215)                  */
CLD bool s_check_tuple(const StreamS &T, unsigned pi, const uint32_t *idx) {
    const cl_pattern &p = T.P->pb.p[pi];
    const unsigned nt = p.n_templates;
    for (unsigned t = 0; t < nt; t++) if (!s_match_local(T, p.t[t], T.hdr[idx[t]], idx[t])) return false;
    const SPat &tp = T.P->pat[pi];
    for (unsigned q = 0; q < tp.n_mpairs; q++) {
        const uint8_t *m = tp.mpair[q];
        if (T.fs.ms[T.hdr[idx[m[0]]].modset].first[m[1]] != T.fs.ms[T.hdr[idx[m[2]]].modset].first[m[3]]) return false;
    }
    for (unsigned q = 0; q < tp.n_pairs; q++) {
        const uint8_t *m = tp.pair[q];
        const uint32_t ia = idx[m[0]], ib = idx[m[2]];
        if (!s_key_equal(T, s_slot(T, ia, has_guard(T.hdr[ia]) + m[1]), s_slot(T, ib, has_guard(T.hdr[ib]) + m[3]))) return false;
    }
    if (nt == 1) return true;
    if (nt == 2) return s_linked(T, idx[0], idx[1]);
    const unsigned e = (unsigned)s_linked(T, idx[0], idx[1]) + (unsigned)s_linked(T, idx[0], idx[2]);
    if (e == 2) return true;
    if (e == 0) return false;
    return s_linked(T, idx[1], idx[2]);
}

/* one (pattern, anchor) item of match_patterns (patterns.py:181-216), join form
 * (see match_block in core.cuh); positions are stream positions                */
CLF void s_try_anchor(StreamS &T, unsigned table, uint32_t i, unsigned pi, uint32_t f) {
    const cl_pattern &p = T.P->pb.p[pi];
    const unsigned nt = p.n_templates;
    const uint32_t b = T.bidx[i], lo = T.bo[b], hi = T.bo[b + 1], V = T.cap.V;
    uint32_t idx[3] = { NONE32, NONE32, NONE32 };
    idx[p.join_order[0]] = i;
    for (unsigned k = 1; k < nt; k++) {
        const unsigned t = p.join_order[k], from = p.join_from[k];
        const cl_hdr hf = T.hdr[idx[from]];
        const cl_template &tf = p.t[from];
        if (hf.n_defs != tf.n_defs || hf.n_aux != tf.n_aux || hf.n_uses != tf.n_uses || (hf.flags & CL_IF_EXT)) return;
        const unsigned long long mm = T.fs.ms[hf.modset].mask;
        if ((mm & tf.mods_all) != tf.mods_all || (mm & tf.mods_none)) return;
        const opnd o = s_slot(T, idx[from], has_guard(hf) + p.join_slot[k]);
        if (!is_value(o)) {
            const unsigned ko = kind_of(o.tag);       /* a non-SSA link: the literal product decides */
            if (ko == CL_K_RZ || ko == CL_K_URZ || ko == CL_K_PRED) sf_fail(T, f, CLS_REDO + 1);
            return;
        }
        const uint32_t dp = o.pay < V ? T.defpos[o.pay] : NONE32;
        if (dp == NONE32 || dp < lo || dp >= hi || T.hdr[dp].op != p.t[t].op) return;
        idx[t] = dp;
    }
    if (nt > 1 && !(idx[0] < idx[1] && (nt < 3 || idx[1] < idx[2]))) return;
    /* budget (G1): rank of the tuple in itertools.product order, needed only when the
     * product of the candidate-list sizes can exceed it                             */
    if (hi - lo >= CLS_BIG_BLOCK) {
        uint32_t cn[3] = { 1, 1, 1 };
        int cl[3] = { 0, 0, 0 };
        for (unsigned t = 0; t < nt; t++) { cl[t] = s_class_of(T, table, p.t[t].op); cn[t] = T.ccnt[b][cl[t]]; }
        const unsigned long long prod = (unsigned long long)cn[0] * cn[1] * cn[2];
        if (prod > T.P->pb.budget) {
            unsigned long long r = 0;
            for (unsigned t = 0; t < nt; t++) {
                const uint32_t ci = T.outpos[idx[t]] - T.cbase[b][cl[t]];      /* index inside its candidate list (s_match) */
                r = t == 0 ? ci : r * cn[t] + ci;
            }
            if (r >= T.P->pb.budget) return;
        }
    }
    if (!s_check_tuple(T, pi, idx)) return;
    const uint32_t m = a_inc_agg(&T.n_mt);
    if (m < T.cap.M) {
        SMatch r;
        r.pat = (uint8_t)pi; r.n = (uint8_t)nt; r.pad = 0;
        r.pos[0] = idx[0]; r.pos[1] = nt > 1 ? idx[1] : NONE32; r.pos[2] = nt > 2 ? idx[2] : NONE32;
        T.mt[m] = r;
        T.mstate[m] = MS_UNDECIDED;
    } else
        s_fail(T);
    a_add(&T.f_stats[f][pi], 1u);
}

template <class G> CLF void s_match(const G &g, StreamS &T, unsigned table) {
    const uint32_t n = T.n, nb = T.nb;
    /* class counts only where a candidate product can reach the budget */
    SFOR(g, b, nb) {
        T.b_over[b] = 0;
        if (T.bo[b + 1] - T.bo[b] >= CLS_BIG_BLOCK) for (int c = 0; c < MAX_CLS; c++) T.ccnt[b][c] = 0;
    }
    if (g.rank == 0) { T.n_mt = 0; T.n_items = 0; }
    g.sync();
    /* seed classes (FindSeeds) */
    SFOR(g, i, n) {
        int c = -1;
        const uint32_t f = T.fidx[i];
        if (T.f_gate[f]) {
            c = s_class_of(T, table, T.hdr[i].op);
            if (c >= 0) {
                const uint32_t b = T.bidx[i];
                if (T.bo[b + 1] - T.bo[b] >= CLS_BIG_BLOCK) a_add(&T.ccnt[b][c], 1u);
                if (sf_ok(T, f) && T.P->anchor_mask[table][c] && T.f_odd[f]) sf_fail(T, f, CLS_REDO + 2);
            }
        }
        T.clsid[i] = (uint8_t)c;
    }
    g.sync();
    s_mark(g, T, SP_SEED);
    /* the dense list of (anchor, pattern) work items, in stream order */
    unsigned long long *items = T.owner;                   /* [I]: free until s_select */
    auto mask_of = [&](uint32_t i) -> uint32_t {
        const uint8_t c = T.clsid[i];
        if (c == 0xFF) return 0u;
        const uint32_t pm = T.P->anchor_mask[table][c];
        return pm && sf_ok(T, T.fidx[i]) ? pm : 0u;
    };
    const uint32_t cap_items = T.cap.I;
    const uint32_t n_items = s_scan(g, n, [&](uint32_t i) {
            uint32_t pm = mask_of(i), cnt = 0;
            for (; pm; pm &= pm - 1) cnt++;
            return cnt;
        }, [&](uint32_t i, uint32_t x) {
            uint32_t pm = mask_of(i);
            for (unsigned pi = 0; pm; pi++, pm >>= 1) if (pm & 1u) { if (x < cap_items) items[x] = (unsigned long long)pi << 32 | i; x++; }
        });
    if (n_items > cap_items) { if (g.rank == 0) s_fail(T); g.sync(); return; }
    if (g.rank == 0) T.n_items = n_items;
    s_mark(g, T, SP_ITEMS);
    /* budget (G1): where the product of the candidate-list sizes of a pattern exceeds it, a tuple counts only
     * if its rank in itertools.product order is below it; the rank needs every member's index inside its
     * candidate list = members of its class before it in the block: one stream-wide scan per class concerned */
    {
        uint32_t need = 0;
        SFOR(g, b, nb) {
            if (T.bo[b + 1] - T.bo[b] < CLS_BIG_BLOCK) continue;
            uint32_t m = 0;
            for (unsigned pi = 0; pi < T.P->pb.n_patterns; pi++) {
                const cl_pattern &p = T.P->pb.p[pi];
                if (p.table != table) continue;
                unsigned long long prod = 1;
                uint32_t cm = 0;
                for (unsigned t = 0; t < p.n_templates; t++) { const int c = s_class_of(T, table, p.t[t].op); prod *= T.ccnt[b][c]; cm |= 1u << c; }
                if (prod > T.P->pb.budget) m |= cm;
            }
            T.b_over[b] = (uint16_t)m;
            need |= m;
        }
        const uint32_t all_need = g_any_bits(g, need);
        for (unsigned c = 0; c < T.P->n_cls[table]; c++) {
            if (!((all_need >> c) & 1u)) continue;
            s_scan(g, n, [&](uint32_t j) { return (uint32_t)(T.clsid[j] == c); },
                   [&](uint32_t j, uint32_t x) {
                       if (T.clsid[j] == c) T.outpos[j] = x;
                       const uint32_t b = T.bidx[j];
                       if (j == T.bo[b]) T.cbase[b][c] = x;
                   });
        }
    }
    s_mark(g, T, SP_BUDGET);
    SFOR(g, k, n_items) {
        const unsigned long long it = items[k];
        const uint32_t i = (uint32_t)it, f = T.fidx[i];
        if (sf_ok(T, f)) s_try_anchor(T, table, i, (unsigned)(it >> 32), f);
    }
    g.sync();
    s_mark(g, T, SP_UNIFY);
}

/* select_matches (patterns.py:241-252) for all blocks at once; the key orders
 * like the reference's stable sort: (start, -len, pattern, product order) where
 * product order within one pattern and start is position order.  Matches that
 * compete share a block, so block-relative positions (16 bits: s_load hands
 * bigger blocks back) order them.                                              */
CLD unsigned long long s_key(const StreamS &T, const SMatch &m) {
    const uint32_t lo = T.bo[T.bidx[m.pos[0]]];
    const uint32_t p1 = m.n > 1 ? m.pos[1] - lo : 0xFFFFu, p2 = m.n > 2 ? m.pos[2] - lo : 0xFFFFu;
    return (unsigned long long)(m.pos[0] - lo) << 40 | (unsigned long long)(3u - m.n) << 38 | (unsigned long long)m.pat << 32 |
           (unsigned long long)p1 << 16 | p2;
}
template <class G> CLF uint32_t s_select(const G &g, StreamS &T) {
    const uint32_t n = T.n, nm = T.n_mt;
    SFOR(g, p, n) { T.keep[p] = 0; T.sel_at[p] = NONE32; }
    g.sync();
    for (;;) {
        SFOR(g, m, nm) if (T.mstate[m] == MS_UNDECIDED) {
            const SMatch r = T.mt[m];
            bool clash = false;
            for (unsigned t = 0; t < r.n; t++) clash |= T.keep[r.pos[t]] != 0;
            if (clash) T.mstate[m] = MS_REJECTED;
            else for (unsigned t = 0; t < r.n; t++) T.owner[r.pos[t]] = NONE64;
        }
        g.sync();
        SFOR(g, m, nm) if (T.mstate[m] == MS_UNDECIDED) {
            const SMatch r = T.mt[m];
            const unsigned long long key = s_key(T, r);
            for (unsigned t = 0; t < r.n; t++) a_min64(&T.owner[r.pos[t]], key);
        }
        g.sync();
        bool left = false;
        SFOR(g, m, nm) if (T.mstate[m] == MS_UNDECIDED) {
            const SMatch r = T.mt[m];
            const unsigned long long key = s_key(T, r);
            bool mine = true;
            for (unsigned t = 0; t < r.n; t++) mine &= T.owner[r.pos[t]] == key;
            if (mine) {
                T.mstate[m] = MS_SELECTED;
                for (unsigned t = 0; t < r.n; t++) T.keep[r.pos[t]] = 1;      /* keep[] is read again only after the sync */
                T.sel_at[r.pos[0]] = m;
            } else
                left = true;
        }
        if (g.rank == 0) T.iters[0]++;
        if (!g.any(left)) break;
    }
    s_mark(g, T, SP_SELECT);
    const uint32_t capS = T.cap.S;
    const uint32_t count = s_scan(g, n, [&](uint32_t p) { return (uint32_t)(T.sel_at[p] != NONE32); },
        [&](uint32_t p, uint32_t x) {
            if (T.sel_at[p] == NONE32 || x >= capS) return;
            const SMatch m = T.mt[T.sel_at[p]];
            SelRec r;
            r.pat = m.pat; r.n = m.n; r.pad0 = r.pad1 = 0; r.blk = T.bidx[p];
            r.pos[0] = m.pos[0]; r.pos[1] = m.pos[1]; r.pos[2] = m.pos[2];
            T.sel[x] = r;
            a_add(&T.f_stats[T.fidx[p]][16 + m.pat], 1u);
        });
    if (count > capS) { if (g.rank == 0) s_fail(T); g.sync(); return 0; }
    s_mark(g, T, SP_SELSCAN);
    return count;
}

/* fix-up of one staged match once the bases are known: inserted records go to
 * out .. out + nins of the (already permuted) stream                          */
CLF void s_apply_stage(StreamS &T, Stage &st, uint32_t out, uint32_t f, uint32_t blk) {
    const uint32_t V = T.cap.V;
    for (unsigned k = 0; k < st.nv; k++) {
        const uint32_t v = st.vbase + k;
        if (v >= V) continue;
        T.alive[v] = 1; T.origin[v] = CL_ORG_PAIR;
        T.def_iid[v] = st.val_def[k] < 0 ? -1 : (int32_t)(st.ibase + (uint32_t)st.val_def[k]);
    }
    for (unsigned k = 0; k < st.nq; k++) if (st.mbase + k < T.cap.Q) T.imm[st.mbase + k] = st.imm[k];
    if (!st.ok) return;                      /* refused: the allocations above leak (G4) */
    for (unsigned r = 0; r < st.nins; r++) {
        const SRec q = st.rec[r];
        const uint32_t o = out + r;
        cl_hdr h;
        h.iid = st.ibase + q.iid; h.op = q.op; h.modset = q.modset;
        h.n_defs = q.n_defs; h.n_aux = 0; h.n_uses = q.n_uses; h.flags = 0; h.ext = 0;
        T.hdr[o] = h;
        const unsigned ns = (unsigned)q.n_defs + q.n_uses;
        uint16_t tg[8]; uint32_t py[8];
#pragma unroll
        for (unsigned k = 0; k < 8; k++) {
            uint16_t tg_ = k < 4 ? q.tag[k] : (uint16_t)0;
            uint32_t p_ = k < 4 ? q.pay[k] : 0u;
            if (k < ns && (tg_ & CL_T_REL)) {
                p_ += kind_of(tg_) == CL_K_VALUE ? st.vbase : st.mbase;
                tg_ &= (uint16_t)~CL_T_REL;
            }
            tg[k] = tg_; py[k] = p_;
        }
        *(uint4 *)&T.tag[(size_t)o * 8] = *(const uint4 *)tg;
        ((uint4 *)&T.pay[(size_t)o * 8])[0] = ((const uint4 *)py)[0];
        ((uint4 *)&T.pay[(size_t)o * 8])[1] = ((const uint4 *)py)[1];
        T.fidx[o] = f; T.bidx[o] = blk;
    }
    for (unsigned k = 0; k < st.nupd; k++) if (st.upd_vid[k] < V) T.def_iid[st.upd_vid[k]] = (int32_t)(st.ibase + st.upd_iid[k]);
    for (unsigned k = 0; k < st.ndrop; k++) if (st.drop_vid[k] < V) T.alive[st.drop_vid[k]] = 0;
}

/* _apply_patterns (patterns.py:671-707): one round over every gated function.
 * All blocks are rewritten against the def-use snapshot of the round's start;
 * a rewrite that removes a use of a value defined in a *later* block of its
 * function would be seen by that block's escape test in the reference (G5):
 * such functions are redone sequentially.                                   */
template <class G> CLF void s_apply_patterns(const G &g, StreamS &T, unsigned table, uint32_t phase) {
    if (!T.du_ok) s_usecount(g, T);
    s_match(g, T, table);
    const uint32_t call = T.n_apply;
    if (g.rank == 0 && call < 8) { T.rstat[call][1] = T.n_items; T.rstat[call][2] = T.n_mt; T.n_apply = call + 1; }
    if (T.fail || T.n_mt == 0) return;
    const uint32_t ns = s_select(g, T);
    if (g.rank == 0 && call < 8) T.rstat[call][3] = ns;
    if (T.fail || ns == 0) return;
    const uint32_t n = T.n, nf = T.nf, nb = T.nb, V = T.cap.V;
    SFOR(g, p, n) { T.keep[p] = 1; T.inscnt[p] = 0; }
    SFOR(g, f, nf) T.f_first[f] = NONE32;
    SFOR(g, b, nb) T.b_first[b] = NONE32;
    g.sync();
    /* plan: one lane per selected match, once */
    uint32_t *cnt_v = T.outpos, *cnt_i = T.sel_at;             /* [ns] <= [I]: free until the position scan */
    unsigned long long *base = T.owner;                        /* [ns]: vbase | ibase << 32, then qbase      */
    SFOR(g, j, ns) {
        const SelRec m = T.sel[j];
        Stage &st = T.stage[j];
        st.ok = st.rm = st.nins = st.retag = st.nv = st.nq = st.nupd = st.ndrop = 0;
        st.ni = 0;
        const uint32_t f = T.fidx[m.pos[0]];
        if (j == 0 || T.fidx[T.sel[j - 1].pos[0]] != f) T.f_first[f] = j;
        if (j == 0 || T.sel[j - 1].blk != m.blk) T.b_first[m.blk] = j;
        if (sf_ok(T, f)) {
            RW c;
            c.s = &T.fs; c.st = &st; c.n = m.n; c.pat = m.pat; c.overflow = false; c.stw = &T.f_stat[f];
            for (unsigned t = 0; t < m.n; t++) { c.idx[t] = m.pos[t]; c.h[t] = T.hdr[c.idx[t]]; }
            for (unsigned t = m.n; t < 3; t++) c.idx[t] = NONE32;
            st.ok = run_rewrite(c);
            if (c.overflow) sf_fail(T, f, CLS_REDO + 3);
            if (st.ok && st.rm) {
                /* G5: does a removed record use a value defined in a later block of its function? */
                bool hazard = false;
                for (unsigned t = 0; t < m.n; t++) {
                    if (!(st.rm >> t & 1)) continue;
                    s_value_operands(T, c.h[t], c.idx[t], [&](uint32_t v) {
                        const uint32_t dp = v < V ? T.defpos[v] : NONE32;
                        hazard |= dp != NONE32 && T.bidx[dp] > m.blk;
                    });
                }
                if (hazard) sf_fail(T, f, CLS_REDO + 4);
            }
        }
        cnt_v[j] = st.nv; cnt_i[j] = st.ni;
        T.mstate[j] = st.nq;                                   /* [ns] <= [M] */
    }
    g.sync();
    s_mark(g, T, SP_PLAN);
    /* exclusive scans in select order (stream wide; rebased per function below): id bases (G3) */
    s_scan(g, ns, [&](uint32_t j) { return cnt_v[j]; }, [&](uint32_t j, uint32_t x) { base[j] = x; });
    s_scan(g, ns, [&](uint32_t j) { return cnt_i[j]; }, [&](uint32_t j, uint32_t x) { base[j] |= (unsigned long long)x << 32; });
    s_scan(g, ns, [&](uint32_t j) { return (uint32_t)T.mstate[j]; }, [&](uint32_t j, uint32_t x) { cnt_v[j] = x; });
    SFOR(g, j, ns) {
        const SelRec m = T.sel[j];
        const uint32_t f = T.fidx[m.pos[0]];
        Stage &st = T.stage[j];
        const uint32_t j0 = T.f_first[f];
        const uint32_t rv = (uint32_t)base[j] - (uint32_t)base[j0];
        const uint32_t ri = (uint32_t)(base[j] >> 32) - (uint32_t)(base[j0] >> 32);
        const uint32_t rq = cnt_v[j] - cnt_v[j0];
        st.vbase = T.f_vbase[f] + T.f_nvid[f] + rv; st.ibase = T.f_niid[f] + ri; st.mbase = T.f_qbase[f] + T.f_nimm[f] + rq;
        if (j + 1 == ns || T.fidx[T.sel[j + 1].pos[0]] != f) {
            /* last match of its function: the function's new counters; over its slices -> general kernel */
            if (st.vbase + st.nv > T.f_vbase[f + 1] || st.mbase + st.nq > T.f_qbase[f + 1]) sf_fail(T, f, CLS_REDO + 5);
            T.f_aux[f] = j;
        }
    }
    g.sync();
    s_mark(g, T, SP_BASES);
    SFOR(g, f, nf) if (T.f_first[f] != NONE32 && sf_ok(T, f)) {
        const Stage &st = T.stage[T.f_aux[f]];
        T.f_nvid[f] = st.vbase + st.nv - T.f_vbase[f]; T.f_niid[f] = st.ibase + st.ni; T.f_nimm[f] = st.mbase + st.nq - T.f_qbase[f];
    }
    /* marks, in-place retags (_rw_imad_wide :414-418), diagnostics, counters */
    SFOR(g, j, ns) {
        const SelRec m = T.sel[j];
        const uint32_t f = T.fidx[m.pos[0]];
        if (!sf_ok(T, f)) continue;
        Stage &st = T.stage[j];
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
            s_event(T, f, phase << 28 | (m.blk - T.f_b0[f]), CL_EV_REFUSED, j - T.b_first[m.blk], m.pat, T.blk[m.blk].bid);
        }
    }
    g.sync();
    /* output position of every record (dead functions keep their records as they are) */
    const uint32_t tot = s_scan(g, n, [&](uint32_t p) { return (uint32_t)T.keep[p] + T.inscnt[p]; },
                                [&](uint32_t p, uint32_t x) { T.outpos[p] = x; });
    if (tot > T.cap.I) { if (g.rank == 0) s_fail(T); g.sync(); return; }
    s_mark(g, T, SP_MARK);
    s_permute(g, T, n, [&](uint32_t p) { return T.keep[p] ? T.outpos[p] + T.inscnt[p] : NONE32; });
    s_mark(g, T, SP_PERMUTE);
    /* staged records to their place, value table, immediates */
    SFOR(g, j, ns) {
        const SelRec m = T.sel[j];
        const uint32_t f = T.fidx2[m.pos[0]];              /* old positions: the buffer the permutation read */
        if (!sf_ok(T, f)) continue;
        s_apply_stage(T, T.stage[j], T.outpos[m.pos[m.n - 1]], f, m.blk);
    }
    g.sync();
    s_rebase_blocks(g, T, n, tot);
    s_mark(g, T, SP_STAGE);
    s_usecount(g, T);                        /* for simplify_packs / remove_dead_pseudo of this round */
}

/* ordered compaction of the stream by keep[]                                   */
template <class G> CLF void s_compact(const G &g, StreamS &T) {
    const uint32_t n = T.n;
    const uint32_t tot = s_scan(g, n, [&](uint32_t p) { return (uint32_t)T.keep[p]; }, [&](uint32_t p, uint32_t x) { T.outpos[p] = x; });
    s_permute(g, T, n, [&](uint32_t p) { return T.keep[p] ? T.outpos[p] : NONE32; });
    s_rebase_blocks(g, T, n, tot);
}

/* remove_dead_pseudo (patterns.py:771-791) for the functions with f_gate set.  The first sweep visits the
 * records; pure records that survive it are the only ones that can still die: later rounds of the fixpoint
 * walk that list                                                                                            */
template <class G> CLF void s_dce(const G &g, StreamS &T) {
    if (!T.du_ok) s_usecount(g, T);
    const uint32_t n = T.n, V = T.cap.V;
    uint32_t *list = (uint32_t *)T.owner;                 /* [<= n] <= [2 I] */
    if (g.rank == 0) T.n_items = 0;
    g.sync();
    auto try_kill = [&](uint32_t i, const cl_hdr &h) -> bool {
        unsigned nd = 0; bool used = false;
        s_value_defs(T, h, i, [&](uint32_t v) { nd++; used |= v < V && *(volatile uint32_t *)&T.usecnt[v] != 0; });
        if (!nd) return true;                               /* never dies: not a candidate either */
        if (used) return false;
        T.keep[i] = 0;
        s_value_defs(T, h, i, [&](uint32_t v) { if (v < V) T.alive[v] = 0; });
        s_value_operands(T, h, i, [&](uint32_t v) { if (v < V) a_sub(&T.usecnt[v], 1u); });
        return true;
    };
    uint32_t mine = 0;
    SFOR(g, i, n) {
        T.keep[i] = 1;
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        if (h.op >= CL_OP__COUNT || !(T.fs.opflags[h.op] & CL_OPF_PURE)) continue;
        if (try_kill(i, h)) mine += T.keep[i] == 0;
        else list[a_inc_agg(&T.n_items)] = i;
    }
    uint32_t removed = 0;
    for (;;) {
        const uint32_t dead = g.sum(mine);
        if (g.rank == 0) T.iters[1]++;
        if (!dead) break;
        removed += dead;
        mine = 0;
        const uint32_t nl = T.n_items;
        SFOR(g, k, nl) {
            const uint32_t i = list[k];
            if (!T.keep[i] || !sf_ok(T, T.fidx[i])) continue;
            if (try_kill(i, T.hdr[i])) mine++;
        }
    }
    if (removed) s_compact(g, T);
    s_mark(g, T, SP_DCE);
}

/* simplify_packs + _redirect_values (patterns.py:710-764) for the gated functions;
 * f_red[f] = redirects of function f                                          */
CLD uint32_t s_final_of(const StreamS &T, uint32_t v) {
    while (v < T.cap.V && T.redirect[v] != NONE32) v = T.redirect[v];
    return v;
}
template <class G> CLF void s_simplify(const G &g, StreamS &T) {
    const FS &s = T.fs;
    if (!T.du_ok) s_usecount(g, T);
    const uint32_t n = T.n, nf = T.nf, nb = T.nb, V = T.cap.V;
    WFOR(g, f, nf) {
        if (g_lane(g) == 0) T.f_red[f] = 0;
        if (!sf_on(T, f)) continue;
        const uint32_t vb = T.f_vbase[f], room = T.f_vbase[f + 1] - vb;
        LFOR(g, v, room) T.redirect[vb + v] = NONE32;
    }
    g.sync();
    uint32_t mine = 0;
    SFOR(g, i, n) {
        const cl_hdr h = T.hdr[i];
        if (h.op != CL_OP_PACK64 || h.n_uses != 2) continue;
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f)) continue;
        const unsigned u0 = use0(h);
        const opnd lo = s_slot(T, i, u0), hi = s_slot(T, i, u0 + 1);
        if (!is_value(lo) || !is_value(hi)) continue;
        if ((lo.tag | hi.tag) & (CL_T_NEG | CL_T_NOT)) continue;
        if (lo.pay >= V || hi.pay >= V) continue;
        const uint32_t plo = T.defpos[lo.pay], phi = T.defpos[hi.pay];
        if (plo == NONE32 || phi == NONE32) continue;
        const cl_hdr dlo = T.hdr[plo], dhi = T.hdr[phi];
        if (!(dlo.op == CL_OP_UNPACK64 && has_mod(s, dlo, CL_MB_LO) && dhi.op == CL_OP_UNPACK64 && has_mod(s, dhi, CL_MB_HI))) continue;
        if (!dlo.n_uses || !dhi.n_uses) { sf_fail(T, f, CLS_REDO + 6); continue; }
        const opnd slo = s_slot(T, plo, use0(dlo)), shi = s_slot(T, phi, use0(dhi));
        if (!(is_value(slo) && is_value(shi) && slo.pay == shi.pay)) continue;
        if (!h.n_defs) { sf_fail(T, f, CLS_REDO + 7); continue; }
        const opnd d = s_slot(T, i, def0(h));
        if (!is_value(d)) { sf_fail(T, f, CLS_REDO + 8); continue; }
        if (d.pay < V) T.redirect[d.pay] = slo.pay;
        a_add(&T.f_red[f], 1u);
        mine++;
    }
    const uint32_t changed = g.sum(mine);
    if (!changed) { s_mark(g, T, SP_SIMPLIFY); return; }
    /* the use counts follow the redirects (every use site of the old value becomes one of the new) */
    auto move_use = [&](uint32_t v) {
        const uint32_t fo = s_final_of(T, v);
        if (fo != v && v < V) { a_sub(&T.usecnt[v], 1u); if (fo < V) a_add(&T.usecnt[fo], 1u); }
    };
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_red[f] || !sf_ok(T, f)) continue;
        s_value_operands(T, T.hdr[i], i, move_use);
    }
    SFOR(g, b, nb) {
        const uint32_t f = T.bfun[b];
        if (!T.f_red[f] || !sf_ok(T, f)) continue;
        for (int k = 0; k < 2; k++) if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE) move_use(T.blk[b].term_pay[k]);
    }
    g.sync();
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_red[f] || !sf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) {
            const opnd u = s_slot(T, i, u0 + k);
            if (is_value(u)) { const uint32_t fo = s_final_of(T, u.pay); if (fo != u.pay) T.pay[(size_t)i * 8 + u0 + k] = fo; }
            else if (kind_of(u.tag) == CL_K_MEMREF) {
                cl_memref &m = T.mem[u.pay];
                if (kind_of(m.base_tag) == CL_K_VALUE) m.base_pay = s_final_of(T, m.base_pay);
                if (kind_of(m.ureg_tag) == CL_K_VALUE) m.ureg_pay = s_final_of(T, m.ureg_pay);
            }
        }
        if (has_guard(h)) { const opnd gd = s_slot(T, i, 0); if (is_value(gd)) T.pay[(size_t)i * 8] = s_final_of(T, gd.pay); }
    }
    SFOR(g, b, nb) {
        const uint32_t f = T.bfun[b];
        if (!T.f_red[f] || !sf_ok(T, f)) continue;
        for (int k = 0; k < 2; k++)
            if (kind_of(T.blk[b].term_tag[k]) == CL_K_VALUE) T.blk[b].term_pay[k] = s_final_of(T, T.blk[b].term_pay[k]);
    }
    g.sync();
    s_mark(g, T, SP_SIMPLIFY);
}

/* tag_cuda_objects (patterns.py:895-916)                                      */
template <class G> CLF void s_tag(const G &g, StreamS &T) {
    const FS &s = T.fs;
    const uint32_t n = T.n;
    SFOR(g, i, n) {
        cl_hdr h = T.hdr[i];
        if (h.op != CL_OP_BAR && h.op != CL_OP_WARPSYNC && h.op != CL_OP_SHFL) continue;
        if (!sf_ok(T, T.fidx[i])) continue;
        unsigned kind = 0, use = 7;
        const unsigned u0 = use0(h);
        if (h.op == CL_OP_BAR) {
            if (has_mod(s, h, CL_MB_SYNC)) {
                kind = 1;
                for (unsigned k = 0; k < h.n_uses && k < 7; k++) if (is_imm(s_slot(T, i, u0 + k))) use = k;
            }
        } else if (h.op == CL_OP_WARPSYNC) {
            for (unsigned k = 0; k < h.n_uses && k < 7; k++) {
                const opnd u = s_slot(T, i, u0 + k);
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
/* normalize_reciprocal (patterns.py:817-888), chains in parallel; see tile.cuh
 * for the argument.  Only functions that hold a MUFU.RCP fed by an I2F take
 * part (f_gate).                                                              */
enum { SRF_R0 = 1, SRF_R1 = 2, SRF_R2 = 4, SRF_R3 = 8, SRF_SEED = 16, SRF_Q = 32, SRF_MUFU = 128 };
template <class G> CLF void s_reciprocal(const G &g, StreamS &T) {
    const FS &s = T.fs;
    const uint32_t n = T.n, nf = T.nf, V = T.cap.V;
    SFOR(g, f, nf) { T.f_aux[f] = 0; T.f_gate[f] = 0; }
    if (g.rank == 0) T.n_chain = 0;
    g.sync();
    /* only functions that hold a MUFU.RCP take part */
    bool mine = false;
    SFOR(g, i, n) {
        const cl_hdr h = T.hdr[i];
        if (h.op != CL_OP_MUFU || !has_mod(s, h, CL_MB_RCP) || !h.n_uses) continue;
        const uint32_t f = T.fidx[i];
        if (sf_ok(T, f)) { T.f_gate[f] = 1; mine = true; }
    }
    if (!g.any(mine)) return;
    s_usecount(g, T);
    /* R_0 and the MUFU.RCP records fed by an I2F */
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_gate[f]) continue;
        const cl_hdr h = T.hdr[i];
        uint8_t fl = h.op == CL_OP_F2I ? (uint8_t)(SRF_R0 | SRF_R1 | SRF_R2 | SRF_R3) : (uint8_t)0;
        if (h.op == CL_OP_MUFU && sf_ok(T, f) && has_mod(s, h, CL_MB_RCP) && h.n_uses) {
            const opnd src = s_slot(T, i, use0(h));
            if (is_value(src) && src.pay < V) {
                const uint32_t dp = T.defpos[src.pay];
                if (dp != NONE32 && T.hdr[dp].op == CL_OP_I2F) {
                    if (!h.n_defs || !is_value(s_slot(T, i, def0(h)))) sf_fail(T, f, CLS_REDO + 9);   /* IndexError / AttributeError */
                    else fl |= SRF_MUFU;
                }
            }
        }
        T.flag[i] = fl;
    }
    uint32_t *valbits = T.redirect;
    WFOR(g, f, nf) {
        if (!T.f_gate[f]) continue;
        const uint32_t vb = T.f_vbase[f], room = T.f_vbase[f + 1] - vb;
        LFOR(g, v, room) valbits[vb + v] = 0;
    }
    g.sync();
    for (unsigned k = 1; k <= 3; k++) {
        const uint8_t prev = (uint8_t)(1u << (k - 1)), cur = (uint8_t)(1u << k);
        SFOR(g, i, n) if (T.flag[i] & prev) {
            const uint32_t f = T.fidx[i];
            if (!sf_on(T, f)) continue;
            s_value_operands(T, T.hdr[i], i, [&](uint32_t v) { if (v < V) valbits[v] |= cur; });
        }
        g.sync();
        SFOR(g, i, n) if (!(T.flag[i] & cur)) {
            const uint32_t f = T.fidx[i];
            if (!sf_on(T, f)) continue;
            bool r = false;
            s_value_defs(T, T.hdr[i], i, [&](uint32_t v) { r |= v < V && (valbits[v] & cur); });
            if (r) T.flag[i] |= (uint8_t)((0xFu << k) & 0xFu);        /* R_k implies R_k+1.. */
        }
        g.sync();
    }
    /* accepted chains */
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        if (h.op != CL_OP_IADD && h.op != CL_OP_IADD3) continue;
        bool any_imm = false;
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) any_imm |= is_imm(s_slot(T, i, u0 + k));
        if (!any_imm) continue;
        unsigned hits = 0;
        uint32_t mp = NONE32, rcp = 0;
        s_value_operands(T, h, i, [&](uint32_t v) {
            const uint32_t dp = v < V ? T.defpos[v] : NONE32;
            if (dp == NONE32 || !(T.flag[dp] & SRF_MUFU)) return;
            const opnd d0 = s_slot(T, dp, def0(T.hdr[dp]));
            if (!is_value(d0) || d0.pay != v) return;
            hits++; mp = dp; rcp = v;
        });
        if (!hits) continue;
        if (hits > 1 || has_guard(h) || (h.flags & CL_IF_EXT)) { sf_fail(T, f, CLS_REDO + 10); continue; }
        if (!(T.flag[i] & SRF_R3)) continue;
        if (T.bidx[mp] != T.bidx[i] || !h.n_defs || !is_value(s_slot(T, i, def0(h)))) { sf_fail(T, f, CLS_REDO + 11); continue; }
        const uint32_t c = a_inc_agg(&T.n_chain);
        if (c < T.cap.X) {
            SChain ch;
            ch.add = i; ch.mufu = mp; ch.rcp = rcp; ch.addv = s_slot(T, i, def0(h)).pay; ch.f = f; ch.rank = 0;
            T.chain[c] = ch;
        } else
            s_fail(T);
        T.flag[i] |= SRF_SEED;
        T.flag[mp] |= SRF_SEED;
    }
    g.sync();
    const uint32_t nc = T.n_chain;
    if (nc == 0 || T.fail) return;
    SFOR(g, i, n) { T.keep[i] = 0; T.inscnt[i] = 0; }
    /* interference (tile.cuh): _reaches_f2i reads the user lists of the records at distance 0..2 of the add it
     * starts from, and a rewritten chain changes the user lists of its MUFU's and its add's results.  Chains are
     * rewritten in (MUFU, add) position order, so chain B can only see a chain A of smaller order whose add or
     * MUFU lies within two def-use hops of B's add.  Orders compare inside one function: positions relative to
     * the function's first record (16 bits, s_load hands bigger functions back).
     * owner[i] = { low: own seed order, high: smallest order reached in one hop }.                          */
    uint32_t *mk1 = T.redirect, *mk2 = T.usecnt;
    WFOR(g, f, nf) {
        if (!T.f_gate[f]) continue;
        const uint32_t vb = T.f_vbase[f], room = T.f_vbase[f + 1] - vb;
        LFOR(g, v, room) { mk1[vb + v] = NONE32; mk2[vb + v] = NONE32; }
    }
    SFOR(g, i, n) if (T.f_gate[T.fidx[i]]) T.owner[i] = NONE64;
    g.sync();
    auto key_of = [&](const SChain &ch) -> uint32_t {
        const uint32_t i0 = T.bo[T.f_b0[ch.f]];
        return (ch.mufu - i0) << 16 | (ch.add - i0);
    };
    SFOR(g, c, nc) {
        const SChain ch = T.chain[c];
        const uint32_t key = key_of(ch);
        a_min32((uint32_t *)&T.owner[ch.add], key);           /* little endian: the low word */
        a_min32((uint32_t *)&T.owner[ch.mufu], key);
    }
    g.sync();
    SFOR(g, i, n) if (T.flag[i] & SRF_SEED) {
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f)) continue;
        const uint32_t key = (uint32_t)T.owner[i];
        s_value_operands(T, T.hdr[i], i, [&](uint32_t v) { if (v < V) a_min32(&mk1[v], key); });
    }
    g.sync();
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f)) continue;
        uint32_t q1 = NONE32;
        s_value_defs(T, T.hdr[i], i, [&](uint32_t v) { if (v < V && mk1[v] < q1) q1 = mk1[v]; });
        if (q1 != NONE32) T.owner[i] = (T.owner[i] & 0xFFFFFFFFull) | (unsigned long long)q1 << 32;
    }
    g.sync();
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!sf_on(T, f) || T.owner[i] == NONE64) continue;
        const uint32_t own = (uint32_t)T.owner[i], q1 = (uint32_t)(T.owner[i] >> 32);
        const uint32_t key = own < q1 ? own : q1;
        s_value_operands(T, T.hdr[i], i, [&](uint32_t v) { if (v < V) a_min32(&mk2[v], key); });
    }
    g.sync();
    SFOR(g, c, nc) {
        const SChain ch = T.chain[c];
        const uint32_t key = key_of(ch);
        uint32_t q = (uint32_t)(T.owner[ch.add] >> 32);
        s_value_defs(T, T.hdr[ch.add], ch.add, [&](uint32_t v) { if (v < V && mk2[v] < q) q = mk2[v]; });
        if (q < key) T.flag[ch.add] |= SRF_Q;
    }
    g.sync();
    /* rank, ids, value table; vmap (usecnt[]) = add result -> its float view */
    WFOR(g, f, nf) {
        if (!T.f_gate[f]) continue;
        const uint32_t vb = T.f_vbase[f], room = T.f_vbase[f + 1] - vb;
        LFOR(g, v, room) T.usecnt[vb + v] = NONE32;
    }
    /* number of a chain inside its function = chains of earlier MUFUs (scan over the records) + chains of
     * the same MUFU with an earlier add (a short list per MUFU: owner[m] low word = head, SChain.rank = next) */
    SFOR(g, i, n) if (T.f_gate[T.fidx[i]]) T.owner[i] = 0xFFFFFFFFull;        /* high word: chains of this MUFU */
    g.sync();
    SFOR(g, c, nc) {
        SChain &ch = T.chain[c];
        if ((T.flag[ch.add] & SRF_Q) != 0) { sf_fail(T, ch.f, CLS_REDO + 12); continue; }
#if CL_DEV
        ch.rank = atomicExch((uint32_t *)&T.owner[ch.mufu], c);
        atomicAdd((uint32_t *)&T.owner[ch.mufu] + 1, 1u);
#else
        ch.rank = (uint32_t)T.owner[ch.mufu];
        T.owner[ch.mufu] = ((T.owner[ch.mufu] >> 32) + 1) << 32 | c;
#endif
        a_add(&T.f_aux[ch.f], 1u);
    }
    g.sync();
    s_scan(g, n, [&](uint32_t j) { return T.f_gate[T.fidx[j]] ? (uint32_t)(T.owner[j] >> 32) : 0u; },
           [&](uint32_t j, uint32_t x) {
               const uint32_t f = T.fidx[j];
               if (!T.f_gate[f]) return;
               T.outpos[j] = x;
               if (j == T.bo[T.f_b0[f]]) T.f_first[f] = x;
           });
    SFOR(g, c, nc) {
        const SChain ch = T.chain[c];
        if (!sf_ok(T, ch.f)) continue;
        uint32_t within = 0;
        for (uint32_t o = (uint32_t)T.owner[ch.mufu]; o != NONE32; o = T.chain[o].rank)
            within += T.chain[o].add < ch.add;
        T.sel_at[ch.add] = T.outpos[ch.mufu] - T.f_first[ch.f] + within;
    }
    g.sync();
    SFOR(g, c, nc) { SChain &ch = T.chain[c]; if (sf_ok(T, ch.f)) ch.rank = T.sel_at[ch.add]; }
    g.sync();
    SFOR(g, c, nc) {
        const SChain ch = T.chain[c];
        const uint32_t f = ch.f;
        if (!sf_ok(T, f)) continue;
        const uint32_t vb = T.f_vbase[f];
        const uint32_t vi = vb + T.f_nvid[f] + 2u * ch.rank, vf = vi + 1u, iid = T.f_niid[f] + 2u * ch.rank;
        if (vf >= T.f_vbase[f + 1]) { sf_fail(T, f, CLS_REDO + 13); continue; }
        /* _insert_reciprocal_bitcasts :863-888 (origin codes carry function-local vids) */
        T.alive[vi] = 1; T.origin[vi] = CL_ORG_BITS | (ch.rcp - vb); T.def_iid[vi] = (int32_t)iid;
        T.alive[vf] = 1; T.origin[vf] = CL_ORG_F | (ch.addv - vb); T.def_iid[vf] = (int32_t)(iid + 1u);
        const cl_hdr ah = T.hdr[ch.add];
        const unsigned u0 = use0(ah);
        for (unsigned k = 0; k < ah.n_uses; k++) {
            const opnd x = s_slot(T, ch.add, u0 + k);
            if (is_value(x) && x.pay == ch.rcp) T.pay[(size_t)ch.add * 8 + u0 + k] = vi;
        }
        T.usecnt[ch.addv] = vf;
        T.keep[ch.add] = 1; T.inscnt[ch.add] = 1;
        s_event(T, f, 1u << 28, CL_EV_BOUNDARY, ch.rank, ch.rcp - vb, ah.iid);
    }
    g.sync();
    /* every user of an add result (top-level uses only :878-883) reads the float view */
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        if (!T.f_aux[f] || !sf_ok(T, f)) continue;
        const cl_hdr h = T.hdr[i];
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) {
            const opnd x = s_slot(T, i, u0 + k);
            if (is_value(x) && x.pay < V && T.usecnt[x.pay] != NONE32) T.pay[(size_t)i * 8 + u0 + k] = T.usecnt[x.pay];
        }
    }
    g.sync();
    /* materialise the bitcasts: a kept add gets one record before and one after it */
    const uint32_t tot = s_scan(g, n, [&](uint32_t p) { return 1u + T.keep[p] + T.inscnt[p]; },
                                [&](uint32_t p, uint32_t x) { T.outpos[p] = x; });
    if (tot > T.cap.I) { if (g.rank == 0) s_fail(T); g.sync(); return; }
    s_permute(g, T, n, [&](uint32_t p) { return T.outpos[p] + T.keep[p]; });
    SFOR(g, c, nc) {
        const SChain ch = T.chain[c];
        const uint32_t f = ch.f;
        if (!sf_ok(T, f)) continue;
        const uint32_t vi = T.f_vbase[f] + T.f_nvid[f] + 2u * ch.rank, iid = T.f_niid[f] + 2u * ch.rank;
        const uint32_t blk = T.bidx2[ch.add];
        for (unsigned q = 0; q < 2; q++) {
            const uint32_t o = T.outpos[ch.add] + 2u * q;
            cl_hdr h;
            h.iid = iid + q; h.op = CL_OP_BITCAST; h.modset = q ? CL_MS_I2F : CL_MS_F2I;
            h.n_defs = 1; h.n_aux = 0; h.n_uses = 1; h.flags = 0; h.ext = 0;
            T.hdr[o] = h;
            for (unsigned k = 0; k < 8; k++) { T.tag[(size_t)o * 8 + k] = k < 2 ? (uint16_t)CL_K_VALUE : (uint16_t)0; T.pay[(size_t)o * 8 + k] = 0; }
            T.pay[(size_t)o * 8] = vi + q; T.pay[(size_t)o * 8 + 1] = q ? ch.addv : ch.rcp;
            T.fidx[o] = f; T.bidx[o] = blk;
        }
    }
    g.sync();
    SFOR(g, f, nf) if (T.f_aux[f] && sf_ok(T, f)) { T.f_nvid[f] += 2u * T.f_aux[f]; T.f_niid[f] += 2u * T.f_aux[f]; }
    s_rebase_blocks(g, T, n, tot);
}

/* ------------------------------------------------------------ load / store */
/* room a function gets in the corpus-wide value / immediate spaces (host and device agree) */
CLHD uint32_t stream_vcap(uint32_t nvid, uint32_t nrec) { return nvid + nrec + 8; }
CLHD uint32_t stream_qcap(uint32_t nimm, uint32_t nrec) { return nimm + nrec / 2 + 8; }
static constexpr uint32_t CLS_MAX_FUNC = 40000;   /* records: function-relative positions (and growth) stay below 2^16 */

/* rebase the ids of one operand into (in) or out of the corpus-wide index spaces */
CLD uint32_t s_rebase(const StreamS &T, uint32_t f, uint16_t tag, uint32_t pay, bool in) {
    uint32_t d;
    switch (kind_of(tag)) {
    case CL_K_VALUE: d = T.f_vbase[f]; break;
    case CL_K_IMM: d = T.f_qbase[f]; break;
    case CL_K_MEMREF: d = T.f_mbase[f]; break;
    default: return pay;
    }
    return in ? pay + d : pay - d;
}

template <class G> CLF void s_load(const G &g, StreamS &T, const StreamIO &a) {
    const cl_corpus &in = a.in;
    const uint32_t nf = in.n_funcs, nb = in.n_blocks;
    if (g.rank == 0) {
        T.nf = nf; T.nb = nb;
        T.n_ev = 0; T.fail = 0; T.n_chain = 0; T.n_mt = 0; T.n_sel = 0; T.n_items = 0;
    }
    /* functions: slices of the value / immediate spaces by prefix sums of their room */
    SFOR(g, f, nf) {
        const cl_func fn = in.func[f];
        const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1];
        const uint32_t nrec = in.blk_off[b1] - in.blk_off[b0];
        const uint32_t nimm = in.imm_off[f + 1] - in.imm_off[f];
        T.f_arch[f] = fn.arch; T.f_nvid[f] = fn.next_vid; T.f_niid[f] = fn.next_iid;
        T.f_nimm[f] = nimm; T.f_nev[f] = 0; T.f_odd[f] = 0; T.f_nin[f] = nrec;
        T.f_active[f] = 0; T.f_gate[f] = 0; T.f_chg[f] = 0; T.f_red[f] = 0; T.f_aux[f] = 0;
        /* overflow slots, empty functions and very large ones take the general kernel */
        const bool plain = in.ext_off[f + 1] == in.ext_off[f] && b1 > b0 && nrec > 0 && nrec <= CLS_MAX_FUNC;
        T.f_stat[f] = plain ? 0u : CLS_REDO;
    }
    SFOR(g, k, (size_t)nf * 64) (&T.f_stats[0][0])[k] = 0;
    g.sync();
    const uint32_t vtot = s_scan(g, nf, [&](uint32_t f) { return T.f_stat[f] ? 0u : stream_vcap(T.f_nvid[f], T.f_nin[f]); },
                                 [&](uint32_t f, uint32_t x) { T.f_vbase[f] = x; });
    const uint32_t qtot = s_scan(g, nf, [&](uint32_t f) { return T.f_stat[f] ? 0u : stream_qcap(T.f_nimm[f], T.f_nin[f]); },
                                 [&](uint32_t f, uint32_t x) { T.f_qbase[f] = x; });
    if (g.rank == 0) {
        T.f_vbase[nf] = vtot; T.f_qbase[nf] = qtot; T.vtot = vtot; T.qtot = qtot;
        T.n = in.blk_off[nb];
        if (vtot > T.cap.V || qtot > T.cap.Q || T.n > T.cap.I) T.fail = 1;      /* host sizing bug: loud */
    }
    g.sync();
    if (T.fail) return;
    const uint32_t n = T.n;
    /* blocks: one warp per function walks its blocks; records get their function / block index from the block */
    WFOR(g, f, nf) {
        const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1], vb = T.f_vbase[f];
        const bool live = T.f_stat[f] == 0;
        LFOR(g, k, b1 - b0) {
            const uint32_t b = b0 + k;
            T.bfun[b] = f;
            T.bo[b] = in.blk_off[b];
            cl_blk bk = in.blk[b];
            if (live) for (int q = 0; q < 2; q++) if (kind_of(bk.term_tag[q]) == CL_K_VALUE) bk.term_pay[q] += vb;
            T.blk[b] = bk;
        }
        const uint32_t i0 = in.blk_off[b0], i1 = in.blk_off[b1];
        /* block of a record: the blocks of one function are few, walk them */
        uint32_t b = b0;
        for (uint32_t i = i0 + g_lane(g); i < i1; i += g_lanes(g)) {
            while (b + 1 < b1 && in.blk_off[b + 1] <= i) b++;
            T.fidx[i] = f; T.bidx[i] = b;
        }
        /* memrefs: mutable copy in the output, value ids rebased */
        const uint32_t m0 = in.mem_off[f], nm = in.mem_off[f + 1] - m0;
        LFOR(g, m, nm) {
            cl_memref r = in.mem[m0 + m];
            if (live) {
                if (kind_of(r.base_tag) == CL_K_VALUE) r.base_pay += vb;
                if (kind_of(r.ureg_tag) == CL_K_VALUE) r.ureg_pay += vb;
            }
            T.mem[m0 + m] = r;
        }
        if (!live) continue;
        const uint32_t v0 = in.val_off[f], nv = T.f_nvid[f], room = T.f_vbase[f + 1] - vb;
        LFOR(g, v, room) {
            const bool have = v < nv;
            T.alive[vb + v] = have ? in.val_alive[v0 + v] : (uint8_t)0;
            T.def_iid[vb + v] = have ? in.val_def_iid[v0 + v] : -1;
            T.origin[vb + v] = CL_ORG_HOST;
        }
        const uint32_t q0 = in.imm_off[f], nq = T.f_nimm[f], qb = T.f_qbase[f];
        LFOR(g, q, nq) T.imm[qb + q] = in.imm[q0 + q];
    }
    if (g.rank == 0) T.bo[nb] = n;
    g.sync();
    /* records: coalesced; value / immediate / memref ids rebased into the corpus-wide spaces */
    SFOR(g, i, n) {
        const uint32_t f = T.fidx[i];
        *(uint4 *)&T.hdr[i] = *(const uint4 *)(in.hdr + i);
        const uint4 tg4 = *(const uint4 *)(in.tag + (size_t)i * 8);
        uint4 p0 = ((const uint4 *)(in.pay + (size_t)i * 8))[0], p1 = ((const uint4 *)(in.pay + (size_t)i * 8))[1];
        if (T.f_stat[f] == 0) {
            const uint16_t *tags = (const uint16_t *)&tg4;
            uint32_t *pp0 = (uint32_t *)&p0, *pp1 = (uint32_t *)&p1;
#pragma unroll
            for (unsigned k = 0; k < 4; k++) { pp0[k] = s_rebase(T, f, tags[k], pp0[k], true); pp1[k] = s_rebase(T, f, tags[4 + k], pp1[k], true); }
        }
        *(uint4 *)&T.tag[(size_t)i * 8] = tg4;
        ((uint4 *)&T.pay[(size_t)i * 8])[0] = p0;
        ((uint4 *)&T.pay[(size_t)i * 8])[1] = p1;
    }
    g.sync();
}

/* results of the live functions in function order at one reserved place; the others are queued for the
 * general kernel                                                                                       */
template <class G> CLF void s_store(const G &g, StreamS &T, const StreamIO &a) {
    const uint32_t nf = T.nf, n = T.n;
    const bool all_ok = !T.fail;
    auto live = [&](uint32_t f) { return all_ok && T.f_stat[f] == 0; };
    const uint32_t oi = s_scan(g, nf, [&](uint32_t f) { return live(f) ? T.bo[T.f_b0[f + 1]] - T.bo[T.f_b0[f]] : 0u; }, [&](uint32_t f, uint32_t x) { T.f_oi[f] = x; });
    const uint32_t oq = s_scan(g, nf, [&](uint32_t f) { return live(f) ? T.f_nimm[f] : 0u; }, [&](uint32_t f, uint32_t x) { T.f_oq[f] = x; });
    const uint32_t ov = s_scan(g, nf, [&](uint32_t f) { return live(f) ? T.f_nvid[f] : 0u; }, [&](uint32_t f, uint32_t x) { T.f_ov[f] = x; });
    const uint32_t oe = s_scan(g, nf, [&](uint32_t f) { return live(f) ? T.f_nev[f] : 0u; }, [&](uint32_t f, uint32_t x) { T.f_oe[f] = x; });
    if (g.rank == 0) {
        T.res[0] = (uint32_t)a_add64(&a.cursor[0], oi); T.res[1] = (uint32_t)a_add64(&a.cursor[1], oq);
        T.res[2] = (uint32_t)a_add64(&a.cursor[2], ov); T.res[3] = (uint32_t)a_add64(&a.cursor[3], oe);
        const bool fits = (unsigned long long)T.res[0] + oi <= a.cap[0] && (unsigned long long)T.res[1] + oq <= a.cap[1] &&
                          (unsigned long long)T.res[2] + ov <= a.cap[2] && (unsigned long long)T.res[3] + oe <= a.cap[3];
        T.work = fits ? 1u : 0u;
        a_add64(&a.stats[65], oi); a_add64(&a.stats[66], oe);
    }
    g.sync();
    const bool fits = T.work != 0;
    const uint32_t ri = T.res[0], rq = T.res[1], rv = T.res[2], re = T.res[3];
    unsigned long long n_in = 0;
    WFOR(g, f, nf) {
        if (!live(f)) {
            if (g_lane(g) == 0) {
                const uint32_t why = T.f_stat[f] >= CLS_REDO && T.f_stat[f] < CLS_REDO + 23 ? T.f_stat[f] - CLS_REDO : 22u;
                a_add(&T.redo[all_ok ? why : 23u], 1u);
                if (T.f_nin[f] > a.small_max) a.retry_big_list[a_add(a.retry_big_count, 1u)] = f;
                else a.retry_list[a_add(a.retry_count, 1u)] = f;
            }
            continue;
        }
        const uint32_t b0 = T.f_b0[f], b1 = T.f_b0[f + 1], i0 = T.bo[b0], cnt = T.bo[b1] - i0, vb = T.f_vbase[f], qb = T.f_qbase[f];
        if (g_lane(g) == 0) {
            const cl_func fin = a.in.func[f];
            FuncOut o;
            o.f.next_vid = T.f_nvid[f]; o.f.next_iid = T.f_niid[f]; o.f.next_temp_reg = fin.next_temp_reg;
            o.f.arch = fin.arch; o.f.status = (uint8_t)(fits ? CL_ST_OK : CL_ST_CAPACITY); o.f.reserved = 0;
            o.inst_start = ri + T.f_oi[f]; o.n_inst = fits ? cnt : 0; o.imm_start = rq + T.f_oq[f]; o.n_imm = fits ? T.f_nimm[f] : 0;
            o.val_start = rv + T.f_ov[f]; o.ev_start = re + T.f_oe[f]; o.n_ev = fits ? T.f_nev[f] : 0; o.pad = 0;
            a.o_func[f] = o;
            n_in += T.f_nin[f];
            T.f_aux[f] = 0;
        }
        LFOR(g, k, b1 - b0) {
            const uint32_t b = b0 + k;
            cl_blk bk = T.blk[b];
            for (int q = 0; q < 2; q++) bk.term_pay[q] = s_rebase(T, f, bk.term_tag[q], bk.term_pay[q], false);
            a.o_blk[b] = bk;
            a.o_blk_start[b] = fits ? ri + T.f_oi[f] + (T.bo[b] - i0) : 0u;
            a.o_blk_cnt[b] = fits ? T.bo[b + 1] - T.bo[b] : 0u;
        }
        /* memrefs back to function-local value ids */
        const uint32_t m0 = T.f_mbase[f], nm = T.f_mbase[f + 1] - m0;
        LFOR(g, m, nm) {
            cl_memref &r = T.mem[m0 + m];
            if (kind_of(r.base_tag) == CL_K_VALUE) r.base_pay -= vb;
            if (kind_of(r.ureg_tag) == CL_K_VALUE) r.ureg_pay -= vb;
        }
        if (!fits) continue;
        const uint32_t nq = T.f_nimm[f], nv = T.f_nvid[f];
        LFOR(g, q, nq) a.o_imm[(size_t)rq + T.f_oq[f] + q] = T.imm[qb + q];
        LFOR(g, v, nv) {
            const size_t d = (size_t)rv + T.f_ov[f] + v;
            a.o_alive[d] = T.alive[vb + v]; a.o_def_iid[d] = T.def_iid[vb + v]; a.o_origin[d] = T.origin[vb + v];
        }
    }
    if (n_in) a_add64(&a.stats[64], n_in);
    g.sync();
    if (fits) {
        SFOR(g, i, n) {
            const uint32_t f = T.fidx[i];
            if (!live(f)) continue;
            const size_t d = (size_t)ri + T.f_oi[f] + (i - T.bo[T.f_b0[f]]);
            uint4 tg4 = *(const uint4 *)&T.tag[(size_t)i * 8];
            uint4 p0 = ((const uint4 *)&T.pay[(size_t)i * 8])[0], p1 = ((const uint4 *)&T.pay[(size_t)i * 8])[1];
            const uint16_t *tags = (const uint16_t *)&tg4;
            uint32_t *pp0 = (uint32_t *)&p0, *pp1 = (uint32_t *)&p1;
#pragma unroll
            for (unsigned k = 0; k < 4; k++) { pp0[k] = s_rebase(T, f, tags[k], pp0[k], false); pp1[k] = s_rebase(T, f, tags[4 + k], pp1[k], false); }
            *(uint4 *)(a.o_hdr + d) = *(const uint4 *)&T.hdr[i];
            *(uint4 *)(a.o_tag + d * 8) = tg4;
            ((uint4 *)(a.o_pay + d * 8))[0] = p0;
            ((uint4 *)(a.o_pay + d * 8))[1] = p1;
        }
        const uint32_t nev = T.n_ev < T.cap.E ? T.n_ev : T.cap.E;
        SFOR(g, e, nev) {
            const cl_event ev = T.ev[e];
            const uint32_t f = ev.func;
            if (live(f)) a.o_ev[(size_t)re + T.f_oe[f] + a_add(&T.f_aux[f], 1u)] = ev;
        }
    }
    /* match counters of the live functions: a lane's slot is fixed (the group size is a multiple of 64) */
    {
        unsigned long long sum = 0;
        const size_t tot = (size_t)nf * 64;
        for (size_t k = g.rank; k < tot; k += g.size) if (live((uint32_t)(k >> 6))) sum += (&T.f_stats[0][0])[k];
        if (g.size % 64u == 0) { if (sum) a_add64(&a.stats[g.rank & 63u], sum); }
        else for (uint32_t k = 0; k < 64; k++) {             /* one-lane host group */
            unsigned long long s2 = 0;
            for (uint32_t f = 0; f < nf; f++) if (live(f)) s2 += T.f_stats[f][k];
            if (s2) a_add64(&a.stats[k], s2);
        }
    }
    g.sync();
}

/* the four calls of pipeline.py:165-169 on every function of the corpus        */
template <class G> CLF void s_set_gate(const G &g, StreamS &T, int mode) {
    /* 0: live sm52 functions, 1: live active functions, 2: live functions with redirects, 3: all live.
     * Modes 1 and 2 only ever narrow the gate inside the aggregation loop, so use counts stay valid for it;
     * modes 0 and 3 start over.                                                                           */
    const uint32_t nf = T.nf;
    if (g.rank == 0 && (mode == 0 || mode == 3)) T.du_ok = 0;
    SFOR(g, f, nf) {
        bool on = sf_ok(T, f);
        if (mode == 0) on = on && T.f_arch[f] == CL_ARCH_SM52;
        else if (mode == 1) on = on && T.f_active[f];
        else if (mode == 2) on = on && T.f_red[f] != 0;
        T.f_gate[f] = on;
    }
    g.sync();
}
template <class G> CLD bool s_any_gate(const G &g, StreamS &T) {
    bool m = false;
    const uint32_t nf = T.nf;
    SFOR(g, f, nf) m |= T.f_gate[f] != 0;
    return g.any(m);
}

template <class G> CLF void s_run(const G &g, StreamS &T, const StreamIO &a) {
    const uint32_t passes = a.passes, max_rounds = a.max_rounds;
    s_load(g, T, a);
    s_mark(g, T, SP_LOAD);
    const uint32_t nf = T.nf;
    if (!T.fail && (passes & CL_PASS_XMAD)) {
        s_set_gate(g, T, 0);       /* also: du_ok = 0 (the gate widened or changed) */
        if (s_any_gate(g, T)) {
            s_apply_patterns(g, T, 1, 0);
            if (!T.fail) s_dce(g, T);
        }
    }
    s_mark(g, T, SP_GATE);
    if (!T.fail && (passes & CL_PASS_RECIPROCAL)) { s_reciprocal(g, T); s_mark(g, T, SP_RECIP); }
    if (!T.fail && (passes & CL_PASS_AGGREGATE)) {
        SFOR(g, f, nf) T.f_active[f] = 1;
        if (g.rank == 0) T.du_ok = 0;
        g.sync();
        for (uint32_t round = 0; round < max_rounds && !T.fail; round++) {
            s_set_gate(g, T, 1);
            if (!s_any_gate(g, T)) break;
            if (g.rank == 0) T.iters[2]++;
            s_mark(g, T, SP_GATE);
            SFOR(g, f, nf) T.f_chg[f] = 0;
            g.sync();
            s_apply_patterns(g, T, 0, 2 + round);
            if (T.fail) break;
            s_set_gate(g, T, 1);
            s_simplify(g, T);
            s_set_gate(g, T, 2);
            if (s_any_gate(g, T)) s_dce(g, T);
            SFOR(g, f, nf) T.f_active[f] = T.f_active[f] && (T.f_chg[f] + T.f_red[f]) != 0;
            g.sync();
        }
        if (!T.fail) { s_set_gate(g, T, 3); s_dce(g, T); }
    }
    s_mark(g, T, SP_GATE);
    if (!T.fail && (passes & CL_PASS_TAG)) s_tag(g, T);
    g.sync();
    s_mark(g, T, SP_TAG);
    s_store(g, T, a);
    s_mark(g, T, SP_STORE);
}

/* once per launch: seed classes of both tables, anchors, unification constraints */
template <class G> CLF void s_setup(const G &g, StreamP &P, const cl_pattern_blob *pb) {
    {
        const uint32_t *src = (const uint32_t *)pb;
        uint32_t *dst = (uint32_t *)&P.pb;
        SFOR(g, k, sizeof(cl_pattern_blob) / 4) dst[k] = src[k];
        SFOR(g, k, 2 * CL_OP__COUNT) (&P.op_cls[0][0])[k] = 0xFF;
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
    SFOR(g, pi, P.pb.n_patterns) {
        const cl_pattern &p = P.pb.p[pi];
        SPat &tp = P.pat[pi];
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

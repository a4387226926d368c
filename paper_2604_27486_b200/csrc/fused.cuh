/* fused.cuh -- the function-resident form of the post-SSA stage (round 2).
 *
 * One cooperative group (one warp for small functions, two or four warps for
 * larger ones) keeps ONE function resident in shared memory from its load to
 * its store and runs every pass of pipeline.py:165-169 on it there:
 *
 *   normalize_xmad / apply_aggregations   patterns.py:794-810
 *     match_patterns (join form)          :181-216   one lane per anchor record
 *     select_matches                      :241-252   greedy scan as repeated group-min
 *     rewrites                            :324-511   one lane, in the reference's own order
 *     simplify_packs, remove_dead_pseudo  :710-791   redirect sweep, worklist DCE
 *   tag_cuda_objects                      :895-916
 *
 * HBM sees one read of the function and one write of its result.
 *
 * What makes the resident form cheap:
 *   * records never move.  The stream is an arena of record slots plus an
 *     order list (position -> slot); a rewrite appends its new records to the
 *     arena, and one scan per round rebuilds the order list.  The only
 *     permutation of 64-byte records is the final store.
 *   * def-use (use counts, defining slot of every value) is built once and
 *     kept valid by every edit, so no pass rebuilds it; dead-pseudo
 *     elimination is driven by a worklist of the values whose count drops to
 *     zero instead of sweeps to a fixpoint.
 *   * rewrites run in the reference's sequential order (blocks by bid,
 *     matches in select order), with the use counts frozen for the duration
 *     of a block exactly like the reference's per-block def-use snapshot
 *     (patterns.py:674,706): ids come out of plain counters (G3, G4) and the
 *     cross-block escape rule (G5) needs no hazard detection.
 *
 * Anything outside the common case -- overflow slots, reciprocal chains,
 * non-SSA join links, a reference exception, a capacity of the shared-memory
 * slice -- makes the group drop the function untouched and queue it for the
 * general per-function kernel of core.cuh (hand-back), so results are
 * bit-equal to the oracle on every input.
 *
 * Written against a small group interface (FG<NW>) so the same source also
 * compiles with a one-lane group for the CPU debug build under tests/sim.
 */
#pragma once
#include "core.cuh"
#include "kargs.h"
#if !CL_DEV
#include <stdio.h>
#include <stdlib.h>
#endif

namespace clk {

/* --------------------------------------------------- compiled pattern table */
/* Host-derived from cl_pattern_blob by fprog_build (culifter.cu, at
 * cl_set_patterns): per template only the slots that need a test, per pattern
 * the equalities between slots that Bindings.bind enforces (patterns.py:93-97). */
struct FChk { uint64_t imm; uint8_t slot, kind, neg, bitnot, half, pad[3]; };
struct FTmpl {
    uint64_t mods_all, mods_none;
    uint16_t op;
    uint8_t n_defs, n_aux, n_uses, n_chk, n_mv, cls;
    uint8_t mv_group[2], pad[6];
    FChk chk[8];
};
static constexpr int F_MAX_PAIRS = 12;
struct FPat {
    uint8_t nt, rewrite, table, n_pairs, n_mpairs, cond_group, bop_group, pad0;
    uint8_t order[3], from[3], jslot[3];
    uint8_t var_t[3], var_k[3], pad1;      /* CL_RW_XMAD: first slot mentioning $a $b $c */
    uint8_t pair[F_MAX_PAIRS][4];          /* tA, kA, tB, kB (slots in defs, aux, uses order) */
    uint8_t mpair[4][4];                   /* tA, groupA, tB, groupB                          */
    FTmpl t[3];
};
static constexpr int F_OPS = (CL_OP__COUNT + 15) & ~15;
struct FProg {
    uint32_t n_patterns, budget, ok, pad;
    uint32_t n_cls[2];
    uint32_t three[2];                     /* table holds a three-template pattern            */
    uint16_t anchor_mask[2][MAX_CLS];
    uint8_t op_cls[2][F_OPS];              /* opcode id -> seed class of the table, 15 = none */
    uint8_t opflags[F_OPS];
    uint8_t group_pos[64];
    uint16_t isetp64_ms[8][2][8];
    FPat p[CL_MAX_PATTERNS];
};

/* ------------------------------------------------------------------ groups */
/* NW warps of one CTA working on one function.  NW == 1: a warp.  NW > 1: a
 * named barrier per group.  NW == 0: one lane (CPU debug build).            */
template <int NW> struct FG {
    static constexpr uint32_t THREADS = NW * 32;
    uint32_t rank, size, bar;
    uint32_t *red;                         /* [16] words of the group's shared memory (FW::gred) */
#if CL_DEV
    CLD void sync() const {
        if (NW == 1) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NW * 32) : "memory");
    }
    CLD uint32_t exscan(uint32_t x, uint32_t &total) const {
        const uint32_t lane = rank & 31u;
        uint32_t v = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, d); if (lane >= (uint32_t)d) v += t; }
        if (NW == 1) { total = __shfl_sync(0xFFFFFFFFu, v, 31); return v - x; }
        const uint32_t w = rank >> 5;
        if (lane == 31) red[w] = v;
        sync();
        uint32_t pre = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < NW; i++) { const uint32_t t = red[i]; if ((uint32_t)i < w) pre += t; tot += t; }
        sync();
        total = tot;
        return pre + v - x;
    }
    CLD bool any(bool f) const {
        const bool b = __any_sync(0xFFFFFFFFu, f);
        if (NW == 1) return b;
        if ((rank & 31u) == 0) red[rank >> 5] = b;
        sync();
        uint32_t r = 0;
#pragma unroll
        for (int i = 0; i < NW; i++) r |= red[i];
        sync();
        return r != 0;
    }
    CLD unsigned long long min64(unsigned long long x) const {
#pragma unroll
        for (int d = 16; d; d >>= 1) { const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, x, d); if (t < x) x = t; }
        if (NW == 1) return x;
        unsigned long long *r64 = (unsigned long long *)(red + 4);
        if ((rank & 31u) == 0) r64[rank >> 5] = x;
        sync();
        unsigned long long r = r64[0];
#pragma unroll
        for (int i = 1; i < NW; i++) { const unsigned long long t = r64[i]; if (t < r) r = t; }
        sync();
        return r;
    }
#endif
};
template <> struct FG<0> {
    static constexpr uint32_t THREADS = 1;
    uint32_t rank, size, bar;
    uint32_t *red;
    CLMEM void sync() const {}
    CLMEM uint32_t exscan(uint32_t x, uint32_t &total) const { total = x; return 0; }
    CLMEM bool any(bool f) const { return f; }
    CLMEM unsigned long long min64(unsigned long long x) const { return x; }
};

/* uniform strided loop over the lanes of a group (like GFOR of core.cuh), never unrolled: code size is what bounds this stage */
#define FFOR(g, i, n) _Pragma("unroll 1") for (uint32_t _b##i = 0, i = (g).rank; _b##i < (n); _b##i += (g).size, i += (g).size)

/* ------------------------------------------------- work pooled over a CTA */
/* The per-item phases (unify one anchor against one pattern, plan one selected
 * match) have a handful of items per function: run by the function's own group
 * they keep 2-4 of 32 lanes busy.  The groups of a CTA are in lock step anyway,
 * so these phases pool the items of all resident functions, sorted by pattern,
 * and every warp of the CTA takes 32 consecutive ones: full warps running one
 * pattern's code.  Shared by the CTA: items per (group, pattern), their first
 * pooled index.                                                              */
static constexpr int F_MAXG = 16;
struct FCta {
    uint32_t cnt[F_MAXG][CL_MAX_PATTERNS];
    uint32_t base[F_MAXG][CL_MAX_PATTERNS];
    uint32_t pstart[CL_MAX_PATTERNS + 1];
    uint32_t total, pad[2];
};
template <class C> struct FW;
template <class C> struct FCtx {              /* a thread's view of its CTA */
    FCta *Q; uint8_t *w0; uint32_t stride, ng, gi, tid, nthreads;
    CLMEM FW<C> &w(uint32_t g) const { return *(FW<C> *)(w0 + (size_t)g * stride); }
};
CLD void f_cta_sync() {
#if CL_DEV
    __syncthreads();
#endif
}
CLD bool f_cta_or(bool x) {
#if CL_DEV
    return __syncthreads_or(x) != 0;
#else
    return x;
#endif
}
/* pooled index of every (group, pattern) segment, pattern major; the groups wrote their cnt row before */
template <class C> CLF uint32_t f_pool_layout(const FCtx<C> &x) {
    f_cta_sync();
    FCta &Q = *x.Q;
#if CL_DEV
    if (x.tid < 32) {
        const uint32_t pi = x.tid & 15u;
        uint32_t sum = 0;
        if (x.tid < 16) {
#pragma unroll 1
            for (uint32_t g = 0; g < x.ng; g++) sum += Q.cnt[g][pi];
        }
        uint32_t v = sum;
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) { const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, d); if ((x.tid & 31u) >= (uint32_t)d) v += t; }
        if (x.tid < 16) {
            uint32_t run = v - sum;
            Q.pstart[pi] = run;
#pragma unroll 1
            for (uint32_t g = 0; g < x.ng; g++) { Q.base[g][pi] = run; run += Q.cnt[g][pi]; }
            if (pi == 15) { Q.pstart[16] = v; Q.total = v; }
        }
    }
#else
    uint32_t run = 0;
    for (uint32_t pi = 0; pi < 16; pi++) { Q.pstart[pi] = run; for (uint32_t g = 0; g < x.ng; g++) { Q.base[g][pi] = run; run += Q.cnt[g][pi]; } }
    Q.pstart[16] = run; Q.total = run;
#endif
    f_cta_sync();
    return Q.total;
}
/* pooled item i -> pattern, group, index inside the group's segment */
template <class C> CLD void f_pool_item(const FCtx<C> &x, uint32_t i, uint32_t &pi, uint32_t &g, uint32_t &k) {
    const FCta &Q = *x.Q;
    pi = 0;
#pragma unroll 1
    while (pi < 15 && Q.pstart[pi + 1] <= i) pi++;
    g = 0;
#pragma unroll 1
    while (g + 1 < x.ng && Q.base[g + 1][pi] <= i) g++;
    k = i - Q.base[g][pi];
}

/* ------------------------------------------------------- size classes */
/* I: record slots of the arena, IN: largest input the class accepts, V: values,
 * B: blocks, MR: memrefs, Q: new immediates, L: def_iid updates, M: raw matches
 * of one round, E: events (group-private global scratch, not shared memory)  */
struct FCfgS { static constexpr uint32_t I = 128, IN = 104, V = 176, VIN = 144, B = 12, MR = 28, Q = 16, L = 256, M = 48, E = 64, TQ = 24; };
struct FCfgL { static constexpr uint32_t I = 256, IN = 208, V = 352, VIN = 288, B = 24, MR = 56, Q = 32, L = 512, M = 80, E = 128, TQ = 32; };
struct FCfgX { static constexpr uint32_t I = 512, IN = 416, V = 704, VIN = 576, B = 48, MR = 112, Q = 64, L = 1024, M = 192, E = 256, TQ = 96; };

enum { SF_LIVE = 1, SF_PURE = 2, SF_INS = 4 /* waits in an insertion list for the next rebuild */, SF_TAKEN = 8, SF_CLS_SHIFT = 4, SF_NOCLS = 15 };
enum { FF_ODD = 1, FF_RZDEF = 2, FF_PREDDEF = 4, FF_RCP = 8, FF_WLOVER = 16, FF_SWEPT = 32 };
static constexpr uint16_t F_NONE = 0xFFFFu;
static constexpr uint8_t INS_AFTER = 0x80;      /* FW::inscnt: the last inserted record goes after the anchor */
static constexpr uint32_t F_REDO = 100;        /* internal: redo this function on the general kernel */

struct FMatch { uint16_t slot[3]; uint8_t pat, n; };
struct FDLog { uint32_t vid; int32_t iid; };

template <class C> struct FW {                 /* one function resident in a group's shared memory */
    alignas(16) cl_hdr hdr[C::I];
    alignas(16) uint16_t tag[C::I * 8];
    alignas(16) uint32_t pay[C::I * 8];
    alignas(16) cl_imm newimm[C::Q];
    cl_imm timm[C::TQ];                         /* immediates of the rewrites being planned (staged until their index is known) */
    cl_event *ev;                               /* [C::E] events of the function: group-private global scratch */
    FDLog *dlog;                                /* [C::L] def_iid updates in program order: same scratch         */
    const cl_imm *imm_in;                       /* immediates of the resident function (global, read only)      */
    cl_blk blk[C::B];
    cl_memref mem[C::MR];
    uint32_t usecnt[C::V];
    uint32_t ccnt[C::B][MAX_CLS];
    uint32_t acnt[2 * (MAX_CLS + 4)];           /* anchors per seed class, then the fill cursors (f_match) */
    FMatch mt[C::M];
    unsigned long long prof[PF__N], prof_t;   /* cycles per phase (lane 0), flushed at the end of the loop */
    uint32_t fstat[64];
    uint32_t gred[16];                          /* scratch of the group collectives (FG::red) */
    /* scalars (one copy per group; control flow reads them through f_rd: sync, read, sync) */
    uint32_t f, n_in, nb, nv_in, nq_in, n_mem, arch, i0, b0, q0, m0, v0;
    uint32_t n_slots, n_pos, cur, next_vid, next_iid, next_temp, n_newimm, n_log, n_mt, n_sel;
    uint32_t wl_tail, n_ev, fail, dirty, flags, nred, big_blocks, n_mev;
    uint32_t r_inst, r_imm, r_val, r_ev, work, ret, n_free, n_timm;
    uint32_t j0, j1, j_next, pad2;               /* rewrite steps: the block run being rewritten, first match of the next one */
    uint16_t defslot[C::V], redirect[C::V], vtmp[C::V];
    uint16_t norigin[C::V];                     /* ValueInfo.origin of the values created here: kind << 14 | vid (f_origin) */
    uint16_t ord[2][C::I], posof[C::I], insslot[C::I], outpos[C::I], wl[C::I];
    uint16_t nxt[C::I];                         /* next record of an anchor's insertion list */
    uint16_t fre[C::I];                         /* free record slots (of removed records)     */
    uint16_t esc[C::M];                         /* per selected match: which defs of its records escape (bit 4t + k) */
    uint16_t bo[C::B + 2];
    uint16_t sel[C::M];
    alignas(4) uint8_t sflag[C::I];
    uint8_t alive[C::V];
    uint8_t sblk[C::I], inscnt[C::I];
    uint8_t mstate[C::M];
    uint8_t tnext[C::TQ];                       /* next staged immediate of the same match, 0xFF = last */
};

/* what a group needs besides its FW                                          */
struct FEnv {
    const FProg *P;                /* shared memory copy                           */
    const KArgs *a;
    const cl_modset *ms;
};

/* ------------------------------------------------------------ small helpers */
template <class C> CLD void f_fail(FW<C> &W, uint32_t code) { a_cas0(&W.fail, code); }
template <class C> CLD bool f_ok(const FW<C> &W) { return *(volatile const uint32_t *)&W.fail == 0; }
/* a group-shared scalar as a *uniform* control decision: every lane has read it before any lane moves on
 * (a lane running ahead could otherwise change it, the group would split and its barriers mismatch)    */
template <class G> CLD uint32_t f_rd(const G &g, const uint32_t *p) { const uint32_t v = *(volatile const uint32_t *)p; g.sync(); return v; }
template <class G, class C> CLD bool f_oks(const G &g, const FW<C> &W) { return f_rd(g, &W.fail) == 0; }
template <class C> CLD opnd f_slot(const FW<C> &W, uint32_t s, unsigned k) {
    opnd o; o.tag = W.tag[s * 8 + k]; o.pay = W.pay[s * 8 + k];
    return o;
}
template <class C> CLD cl_imm f_imm_at(const FW<C> &W, const FEnv &e, uint32_t idx) {
    (void)e;
    if (idx < W.nq_in) return W.imm_in[idx];
    return W.newimm[(idx - W.nq_in) & (C::Q - 1)];
}
template <class C> CLD bool f_live(const FW<C> &W, uint32_t s) { return (W.sflag[s] & SF_LIVE) != 0; }
/* value_operands (ssa.py:599-610) / all_defs of one record, as a packed list of value ids.
 * Out of line and rolled: every pass asks for them, and the unrolled, inlined form of these
 * loops was most of the kernel's code (the stage is instruction-fetch bound).               */
struct FVals { unsigned long long lo, hi; uint32_t n; };
CLD uint32_t f_val(const FVals &u, uint32_t k) { return (uint32_t)((k < 4 ? u.lo : u.hi) >> ((k & 3u) * 16u)) & 0xFFFFu; }
CLD void f_val_push(FVals &u, uint32_t v) {
    if (v > 0xFFFFu) v = 0xFFFFu;                    /* no such value: callers range-check */
    if (u.n < 4) u.lo |= (unsigned long long)v << (u.n * 16u);
    else if (u.n < 8) u.hi |= (unsigned long long)v << ((u.n - 4u) * 16u);
    u.n++;                                           /* n > 8: more value operands than the list holds (f_index hands the function back) */
}
template <class C> CLN FVals f_uses(const FW<C> &W, uint32_t s) {
    FVals u; u.lo = u.hi = 0; u.n = 0;
    const cl_hdr h = W.hdr[s];
    if (has_guard(h)) { const opnd g = f_slot(W, s, 0); if (is_value(g)) f_val_push(u, g.pay); }
    const unsigned u0 = use0(h), u1 = u0 + h.n_uses;
#pragma unroll 1
    for (unsigned k = u0; k < u1 && k < 8; k++) {
        const opnd o = f_slot(W, s, k);
        if (is_value(o)) f_val_push(u, o.pay);
        else if (kind_of(o.tag) == CL_K_MEMREF) {
            const cl_memref &m = W.mem[o.pay < C::MR ? o.pay : 0];
            if (kind_of(m.base_tag) == CL_K_VALUE) f_val_push(u, m.base_pay);
            if (kind_of(m.ureg_tag) == CL_K_VALUE) f_val_push(u, m.ureg_pay);
        }
    }
    return u;
}
template <class C> CLN FVals f_defs(const FW<C> &W, uint32_t s) {
    FVals u; u.lo = u.hi = 0; u.n = 0;
    const cl_hdr h = W.hdr[s];
    const unsigned d0 = def0(h), d1 = d0 + h.n_defs + h.n_aux;
#pragma unroll 1
    for (unsigned k = d0; k < d1 && k < 8; k++) { const opnd d = f_slot(W, s, k); if (is_value(d)) f_val_push(u, d.pay); }
    return u;
}
template <class C, class F> CLD void f_value_operands(const FW<C> &W, const cl_hdr &, uint32_t s, F fn) {
    const FVals u = f_uses(W, s);
#pragma unroll 1
    for (uint32_t k = 0; k < u.n && k < 8; k++) fn(f_val(u, k));
}
template <class C, class F> CLD void f_value_defs(const FW<C> &W, const cl_hdr &, uint32_t s, F fn) {
    const FVals u = f_defs(W, s);
#pragma unroll 1
    for (uint32_t k = 0; k < u.n && k < 8; k++) fn(f_val(u, k));
}
/* DCE worklist: the defining record of a value whose use count reached zero  */
template <class C> CLD void f_push_wl(FW<C> &W, uint32_t ds) {
    if (ds == F_NONE) return;
    if ((W.sflag[ds] & (SF_LIVE | SF_PURE)) != (SF_LIVE | SF_PURE)) return;
    const uint32_t k = a_add(&W.wl_tail, 1u);
    if (k < C::I) W.wl[k] = (uint16_t)ds;
    else W.flags |= FF_WLOVER;                   /* racing lanes write the same bit */
}
template <class C> CLN void f_dec_use(FW<C> &W, uint32_t v) {
    if (v >= C::V) return;
    if (a_sub(&W.usecnt[v], 1u) == 1u) f_push_wl(W, W.defslot[v]);
}
template <class C> CLD void f_inc_use(FW<C> &W, uint32_t v) { if (v < C::V) a_add(&W.usecnt[v], 1u); }
template <class C> CLD void f_event(FW<C> &W, uint32_t seq, uint32_t kind, uint32_t idx, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    const uint32_t k = a_add(&W.n_ev, 1u);
    if (k < C::E) {
        cl_event e; e.func = W.f; e.seq = seq; e.kind = kind; e.idx = idx; e.a = a; e.b = b; e.c = c; e.d = d;
        W.ev[k] = e;
    } else
        f_fail(W, F_REDO + 42);
}

/* per-phase cycle clock: lane 0 charges the time since the last stamp to `slot` */
template <class G, class C> CLD void f_prof(const G &g, FW<C> &W, int slot) {
#if CL_DEV
    if (g.rank == 0) { const unsigned long long t = clock64(); W.prof[slot] += t - W.prof_t; W.prof_t = t; }
#else
    (void)g; (void)W; (void)slot;
#endif
}

/* ------------------------------------------------------------------- load */
/* false: the function does not fit this size class (nothing was touched)     */
template <class G, class C> CLF bool f_load(const G &g, FW<C> &W, const FEnv &e, uint32_t f) {
    const cl_corpus &in = e.a->in;
    const uint32_t b0 = in.func_blk_off[f], b1 = in.func_blk_off[f + 1];
    const uint32_t i0 = in.blk_off[b0], n = in.blk_off[b1] - i0, nb = b1 - b0;
    const cl_func fn = in.func[f];
    const uint32_t q0 = in.imm_off[f], nq = in.imm_off[f + 1] - q0;
    const uint32_t m0 = in.mem_off[f], nm = in.mem_off[f + 1] - m0;
    const uint32_t v0 = in.val_off[f];
    if (n > C::IN || nb > C::B || fn.next_vid > C::VIN || nm > C::MR) return false;
    g.sync();                                   /* the previous function's store is done */
    if (g.rank == 0) {
        W.f = f; W.n_in = n; W.nb = nb; W.nv_in = fn.next_vid; W.nq_in = nq; W.n_mem = nm; W.arch = fn.arch;
        W.i0 = i0; W.b0 = b0; W.q0 = q0; W.m0 = m0; W.v0 = v0;
        W.n_slots = n; W.n_pos = n; W.cur = 0; W.next_vid = fn.next_vid; W.next_iid = fn.next_iid; W.next_temp = fn.next_temp_reg;
        W.n_newimm = 0; W.n_log = 0; W.n_mt = 0; W.n_sel = 0; W.wl_tail = 0; W.n_ev = 0; W.fail = 0; W.dirty = 0;
        W.flags = 0; W.nred = 0; W.big_blocks = 0; W.n_mev = 0; W.ret = 0; W.n_free = 0; W.n_timm = 0;
        if (in.ext_off[f + 1] != in.ext_off[f] || nb == 0) W.fail = F_REDO + 1;      /* overflow slots: general kernel */
    }
    if (g.rank == 0) W.imm_in = in.imm + q0;
    {
        const uint4 *sh = (const uint4 *)(in.hdr + i0), *st = (const uint4 *)(in.tag + (size_t)i0 * 8), *sp = (const uint4 *)(in.pay + (size_t)i0 * 8);
        uint4 *dh = (uint4 *)W.hdr, *dt = (uint4 *)W.tag, *dp = (uint4 *)W.pay;
        FFOR(g, i, n) if (i < n) { dh[i] = sh[i]; dt[i] = st[i]; }
        FFOR(g, i, 2 * n) if (i < 2 * n) dp[i] = sp[i];
    }
    FFOR(g, b, nb + 1) if (b <= nb) W.bo[b] = (uint16_t)(in.blk_off[b0 + b] - i0);
    FFOR(g, b, nb) if (b < nb) W.blk[b] = in.blk[b0 + b];
    FFOR(g, m, nm) if (m < nm) W.mem[m] = in.mem[m0 + m];
    FFOR(g, v, fn.next_vid) if (v < fn.next_vid) { W.alive[v] = in.val_alive[v0 + v]; W.usecnt[v] = 0; W.defslot[v] = F_NONE; }
    FFOR(g, k, 64) if (k < 64) W.fstat[k] = 0;
    FFOR(g, i, n) if (i < n) { W.ord[0][i] = (uint16_t)i; W.posof[i] = (uint16_t)i; W.inscnt[i] = 0; }
    g.sync();
    return true;
}

/* seed class of an opcode for one table (FindSeeds, patterns.py:189-191)      */
CLD unsigned f_cls(const FProg &P, unsigned table, uint16_t op) { return op < CL_OP__COUNT ? P.op_cls[table][op] : (unsigned)SF_NOCLS; }

/* def-use (ssa.py:613-636) + per-slot flags, once per function               */
template <class G, class C> CLF void f_index(const G &g, FW<C> &W, const FEnv &e, unsigned table) {
    const FProg &P = *e.P;
    const uint32_t n = W.n_in, nb = W.nb;
    uint32_t fl = 0;
    FFOR(g, s, n) if (s < n) {
        const cl_hdr h = W.hdr[s];
        uint32_t lo = 0, hi = nb;                    /* last b with bo[b] <= s */
        while (lo + 1 < hi) { const uint32_t mid = (lo + hi) >> 1; if (W.bo[mid] <= s) lo = mid; else hi = mid; }
        W.sblk[s] = (uint8_t)lo;
        unsigned sf = SF_LIVE | f_cls(P, table, h.op) << SF_CLS_SHIFT;
        if (h.op < CL_OP__COUNT && (P.opflags[h.op] & CL_OPF_PURE)) sf |= SF_PURE;
        W.sflag[s] = (uint8_t)sf;
        if (h.flags & CL_IF_EXT) { fl |= FF_ODD; continue; }
        if (h.op == CL_OP_MUFU && ((e.ms[h.modset].mask >> CL_MB_RCP) & 1u)) fl |= FF_RCP;
        const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
#pragma unroll 1
        for (unsigned k = 0; k < nd; k++) {
            const opnd d = f_slot(W, s, d0 + k);
            const unsigned kd = kind_of(d.tag);
            if (kd == CL_K_VALUE) { if (d.pay < W.nv_in) W.defslot[d.pay] = (uint16_t)s; else fl |= FF_ODD; }
            else if (kd == CL_K_RZ || kd == CL_K_URZ) fl |= FF_RZDEF;
            else if (kd == CL_K_PRED) fl |= FF_PREDDEF;
            else fl |= FF_ODD;
        }
        {
            const FVals u = f_uses(W, s);
            if (u.n > 8) fl |= FF_ODD;                 /* more value operands than FVals holds */
#pragma unroll 1
            for (uint32_t k = 0; k < u.n && k < 8; k++) { const uint32_t v = f_val(u, k); if (v < W.nv_in) a_add(&W.usecnt[v], 1u); else fl |= FF_ODD; }
        }
    }
    FFOR(g, b, nb) if (b < nb)
#pragma unroll 1
        for (int k = 0; k < 2; k++)
            if (kind_of(W.blk[b].term_tag[k]) == CL_K_VALUE) { const uint32_t v = W.blk[b].term_pay[k]; if (v < W.nv_in) a_add(&W.usecnt[v], 1u); else fl |= FF_ODD; }
#if CL_DEV
    if (fl) atomicOr(&W.flags, fl);
#else
    W.flags |= fl;
#endif
    g.sync();
    if (g.rank == 0 && (W.flags & FF_ODD)) f_fail(W, F_REDO + 2);
    g.sync();
}
/* seed classes of the other table                                            */
template <class G, class C> CLF void f_reclass(const G &g, FW<C> &W, const FEnv &e, unsigned table) {
    const FProg &P = *e.P;
    const uint32_t n = W.n_slots;
    FFOR(g, s, n) if (s < n) W.sflag[s] = (uint8_t)((W.sflag[s] & 15u) | f_cls(P, table, W.hdr[s].op) << SF_CLS_SHIFT);
    g.sync();
}

/* ------------------------------------------------------------ order list */
/* positions of the live records after the insertions and removals since the
 * last call: one scan over the old positions (records themselves stay put)   */
template <class G, class C> CLF void f_rebuild(const G &g, FW<C> &W) {
    const uint32_t n = W.n_pos, cur = W.cur;
    const uint16_t *oo = W.ord[cur];
    uint16_t *on = W.ord[cur ^ 1];
    uint32_t run = 0;
    FFOR(g, p, n) {
        uint32_t c = 0, me = 0;
        if (p < n) {
            const uint32_t s = oo[p];
            me = (W.sflag[s] & (SF_LIVE | SF_INS)) == SF_LIVE;       /* a reused slot belongs to its new place */
            c = me;
            if (W.inscnt[p]) for (uint32_t q = W.insslot[p]; q != F_NONE; q = W.nxt[q]) c += f_live(W, q);
        }
        uint32_t tot;
        const uint32_t o = g.exscan(c, tot);
        if (p < n) {
            uint32_t w = run + o;
            W.outpos[p] = (uint16_t)w;
            /* inserted records go before their anchor; with INS_AFTER the last one goes right after it */
            const uint32_t fl = W.inscnt[p], self = oo[p];
            bool placed = !me;
            if (fl) for (uint32_t q = W.insslot[p]; q != F_NONE; q = W.nxt[q]) {
                if ((fl & INS_AFTER) && W.nxt[q] == F_NONE && !placed) { on[w] = (uint16_t)self; W.posof[self] = (uint16_t)w; w++; placed = true; }
                if (f_live(W, q)) { on[w] = (uint16_t)q; W.posof[q] = (uint16_t)w; w++; }
            }
            if (!placed) { on[w] = (uint16_t)self; W.posof[self] = (uint16_t)w; }
        }
        run += tot;
    }
    g.sync();
    uint16_t *nbo = W.sel;                         /* free outside select .. rewrite */
    FFOR(g, b, W.nb + 1) if (b <= W.nb) { const uint32_t old = W.bo[b]; nbo[b] = old < n ? W.outpos[old] : (uint16_t)run; }
    g.sync();
    FFOR(g, b, W.nb + 1) if (b <= W.nb) W.bo[b] = nbo[b];
    const uint32_t nz = run > n ? run : n;
    FFOR(g, p, nz) if (p < nz) { W.inscnt[p] = 0; if (p < run) W.sflag[on[p]] &= (uint8_t)~SF_INS; }
    if (g.rank == 0) { W.n_pos = run; W.cur = cur ^ 1; W.dirty = 0; }
    g.sync();
}

/* ----------------------------------------------------------------- matching */
/* operand_key equality (patterns.py:109-127)                                   */
template <class C> CLN bool f_key_equal(const FW<C> &W, const FEnv &e, opnd a, opnd b) {
    unsigned ka = kind_of(a.tag), kb = kind_of(b.tag);
    if (ka == CL_K_URZ) ka = CL_K_RZ;
    if (kb == CL_K_URZ) kb = CL_K_RZ;
    const bool oa = ka == CL_K_NONE || ka >= CL_K_MEMREF, ob = kb == CL_K_NONE || kb >= CL_K_MEMREF;
    if (oa || ob) {
        if (!(oa && ob)) return false;
        if (a.pay >= C::MR || b.pay >= C::MR) return false;
        const cl_memref &x = W.mem[a.pay], &y = W.mem[b.pay];           /* ("other", str(op)) */
        if (x.base_tag != y.base_tag || x.ureg_tag != y.ureg_tag) return false;
        if (kind_of(x.base_tag) != CL_K_NONE && x.base_pay != y.base_pay) return false;
        if (kind_of(x.ureg_tag) != CL_K_NONE && x.ureg_pay != y.ureg_pay) return false;
        return x.off_hi == y.off_hi && x.off_lo == y.off_lo;
    }
    if (ka != kb) return false;
    if (ka == CL_K_RZ) return true;
    if (ka == CL_K_IMM) return a.pay == b.pay || f_imm_at(W, e, a.pay).bits == f_imm_at(W, e, b.pay).bits;
    return a.pay == b.pay;
}
/* _match_opcode + the slot-local part of _unify (patterns.py:155-178, :130-152) */
template <class C> CLN bool f_match_local(const FW<C> &W, const FEnv &e, const FTmpl &t, const cl_hdr &h, uint32_t s) {
    if (h.op != t.op) return false;
    if (t.n_defs != h.n_defs || t.n_aux != h.n_aux || t.n_uses != h.n_uses) return false;
    const cl_modset &ms = e.ms[h.modset];
    if ((ms.mask & t.mods_all) != t.mods_all) return false;
    if (ms.mask & t.mods_none) return false;
#pragma unroll 1
    for (unsigned k = 0; k < t.n_mv; k++) if (ms.first[t.mv_group[k]] == 0xFF) return false;
    const unsigned g0 = has_guard(h);
#pragma unroll 1
    for (unsigned q = 0; q < t.n_chk; q++) {
        const FChk &c = t.chk[q];
        const opnd o = f_slot(W, s, g0 + c.slot);
        switch (c.kind) {
        case CL_S_RZ: if (!is_zero(o)) return false; break;
        case CL_S_PT:
            if (!(kind_of(o.tag) == CL_K_PRED && o.pay == CL_PT_INDEX)) return false;
            if (c.neg != 0 && o_neg(o) != (c.neg == 2)) return false;
            break;
        case CL_S_IMM: if (!(is_imm(o) && f_imm_at(W, e, o.pay).bits == c.imm)) return false; break;
        case CL_S_VAR:
            if (c.neg && o_neg(o) != (c.neg == 2)) return false;
            if (c.bitnot && o_not(o) != (c.bitnot == 2)) return false;
            if (c.half && o_half(o) != c.half) return false;
            break;
        default: return false;
        }
    }
    return true;
}
/* index of a record inside the candidate list of its class (patterns.py:190):
 * live records of the class before it in its block                          */
template <class C> CLN uint32_t f_class_rank(const FW<C> &W, uint32_t s) {
    const uint32_t b = W.sblk[s], cls = W.sflag[s] >> SF_CLS_SHIFT, p1 = W.posof[s];
    const uint16_t *o = W.ord[W.cur];
    uint32_t r = 0;
#pragma unroll 1
    for (uint32_t p = W.bo[b]; p < p1; p++) { const uint32_t q = o[p]; r += (W.sflag[q] & SF_LIVE) && (uint32_t)(W.sflag[q] >> SF_CLS_SHIFT) == cls; }
    return r;
}
/* one (pattern, anchor) item of match_patterns (patterns.py:181-216), join form:
 * every other instruction of the tuple is the SSA definition of the operand that
 * links it to an already resolved one, so the candidate product collapses to one
 * tuple per anchor; the tuple's rank in itertools.product order still decides the
 * budget cut (G1).  Def-use connectivity (_connected :219) holds by construction:
 * every member shares its link value with the member it was resolved from.      */
template <class C> CLF void f_try_anchor(FW<C> &W, const FEnv &e, uint32_t s, unsigned pi) {
    const FPat &p = e.P->p[pi];
    const unsigned nt = p.nt;
    uint32_t idx[3] = { s, s, s };
    cl_hdr h[3];
    const unsigned ta = p.order[0];
    h[ta] = W.hdr[s];
    if (!f_match_local(W, e, p.t[ta], h[ta], s)) return;
    const uint32_t blk = W.sblk[s];
#pragma unroll 1
    for (unsigned k = 1; k < nt; k++) {
        const unsigned t = p.order[k], from = p.from[k];
        const opnd o = f_slot(W, idx[from], has_guard(h[from]) + p.jslot[k]);
        if (!is_value(o)) {
            /* a non-SSA link (RZ, PT, a physical predicate) can only equal a def operand of the same kind:
             * if the function has such defs the literal product decides                              */
            const unsigned ko = kind_of(o.tag);
            if (((ko == CL_K_RZ || ko == CL_K_URZ) && (W.flags & FF_RZDEF)) || (ko == CL_K_PRED && (W.flags & FF_PREDDEF))) f_fail(W, F_REDO + 3);
            return;
        }
        const uint32_t dp = o.pay < C::V ? W.defslot[o.pay] : (uint32_t)F_NONE;
        if (dp == F_NONE || !f_live(W, dp) || W.sblk[dp] != blk) return;
        h[t] = W.hdr[dp];
        if (!f_match_local(W, e, p.t[t], h[t], dp)) return;
        idx[t] = dp;
    }
    if (nt > 1 && !(W.posof[idx[0]] < W.posof[idx[1]] && (nt < 3 || W.posof[idx[1]] < W.posof[idx[2]]))) return;
#pragma unroll 1
    for (unsigned q = 0; q < p.n_mpairs; q++) {
        const uint8_t *m = p.mpair[q];
        if (e.ms[h[m[0]].modset].first[m[1]] != e.ms[h[m[2]].modset].first[m[3]]) return;
    }
#pragma unroll 1
    for (unsigned q = 0; q < p.n_pairs; q++) {
        const uint8_t *m = p.pair[q];
        if (!f_key_equal(W, e, f_slot(W, idx[m[0]], has_guard(h[m[0]]) + m[1]), f_slot(W, idx[m[2]], has_guard(h[m[2]]) + m[3]))) return;
    }
    /* budget (G1): only where the product of the candidate-list sizes can exceed it */
    if (W.big_blocks && nt > 1) {
        unsigned long long prod = 1;
#pragma unroll 1
        for (unsigned t = 0; t < nt; t++) prod *= W.ccnt[blk][p.t[t].cls];
        if (prod > e.P->budget) {
            unsigned long long r = 0;
#pragma unroll 1
            for (unsigned t = 0; t < nt; t++) r = (t ? r * W.ccnt[blk][p.t[t].cls] : 0ull) + f_class_rank(W, idx[t]);
            if (r >= e.P->budget) return;
        }
    }
    const uint32_t m = a_add(&W.n_mt, 1u);
    if (m < C::M) {
        FMatch r;
        r.pat = (uint8_t)pi; r.n = (uint8_t)nt;
        r.slot[0] = (uint16_t)idx[0]; r.slot[1] = (uint16_t)(nt > 1 ? idx[1] : F_NONE); r.slot[2] = (uint16_t)(nt > 2 ? idx[2] : F_NONE);
        W.mt[m] = r;
        W.mstate[m] = MS_UNDECIDED;
    } else
        f_fail(W, F_REDO + 43);
    a_add(&W.fstat[pi], 1u);
}

template <class G, class C> CLF void f_match_prep(const G &g, FW<C> &W, const FEnv &e, const FCtx<C> &x, unsigned table) {
    const FProg &P = *e.P;
    if (g.rank == 0) { W.n_mt = 0; W.n_sel = 0; }
    /* blocks long enough for a candidate product above the budget (37^3 > 50 000): class counts */
    bool big = false;
    FFOR(g, b, W.nb) if (b < W.nb) {
        const uint32_t len = W.bo[b + 1] - W.bo[b];
        big |= (unsigned long long)len * len * (P.three[table] ? len : 1u) > P.budget;
    }
    big = g.any(big);
    if (g.rank == 0) W.big_blocks = big;
    const uint16_t *o = W.ord[W.cur];
    const uint32_t n = W.n_pos;
    if (big) {
        FFOR(g, k, W.nb * MAX_CLS) if (k < W.nb * MAX_CLS) (&W.ccnt[0][0])[k] = 0;
        g.sync();
        FFOR(g, p, n) if (p < n) {
            const uint32_t s = o[p], fl = W.sflag[s];
            if ((fl & SF_LIVE) && (fl >> SF_CLS_SHIFT) != SF_NOCLS) a_add(&W.ccnt[W.sblk[s]][fl >> SF_CLS_SHIFT], 1u);
        }
    }
    /* the anchor records, sorted by seed class (counting sort: count, place), so that the lanes of a group
     * work on the same pattern at the same time: one dense loop per pattern instead of one sparse,
     * divergent sweep over the records (measured: 2.5 of 32 lanes active)                            */
    uint16_t *list = W.outpos;                       /* free between rebuild and simplify */
    FFOR(g, k, 2 * (MAX_CLS + 4)) if (k < 2 * (MAX_CLS + 4)) W.acnt[k] = 0;
    g.sync();
    FFOR(g, p, n) if (p < n) {
        const uint32_t s = o[p], fl = W.sflag[s], c = fl >> SF_CLS_SHIFT;
        if ((fl & SF_LIVE) && c != SF_NOCLS && P.anchor_mask[table][c]) a_add(&W.acnt[c], 1u);
    }
    g.sync();
    uint32_t *fill = W.acnt + MAX_CLS + 4;
    if (g.rank == 0) { uint32_t run = 0; for (unsigned c = 0; c < (unsigned)MAX_CLS; c++) { fill[c] = run; run += W.acnt[c]; } }
    g.sync();
    FFOR(g, p, n) if (p < n) {
        const uint32_t s = o[p], fl = W.sflag[s], c = fl >> SF_CLS_SHIFT;
        if ((fl & SF_LIVE) && c != SF_NOCLS && P.anchor_mask[table][c]) list[a_add(&fill[c], 1u)] = (uint16_t)s;
    }
    g.sync();
    /* this group's row of the CTA's item table: anchors of every pattern of the table */
    FFOR(g, pi, CL_MAX_PATTERNS) if (pi < CL_MAX_PATTERNS)
        x.Q->cnt[x.gi][pi] = pi < P.n_patterns && P.p[pi].table == table ? W.acnt[P.p[pi].t[P.p[pi].order[0]].cls] : 0u;
    g.sync();
}
/* a group that sits this match phase out */
template <class G, class C> CLF void f_match_idle(const G &g, const FCtx<C> &x) {
    FFOR(g, pi, CL_MAX_PATTERNS) if (pi < CL_MAX_PATTERNS) x.Q->cnt[x.gi][pi] = 0;
}
/* unify every (anchor, pattern) item of the CTA's resident functions: all threads of the CTA */
template <class C> CLF void f_match_pooled(const FCtx<C> &x, const FEnv &e) {
    const uint32_t total = f_pool_layout(x);
#pragma unroll 1
    for (uint32_t i = x.tid; i < total; i += x.nthreads) {
        uint32_t pi, gq, k;
        f_pool_item(x, i, pi, gq, k);
        FW<C> &Wq = x.w(gq);
        const FPat &p = e.P->p[pi];
        const uint32_t ac = p.t[p.order[0]].cls, lo = Wq.acnt[MAX_CLS + 4 + ac] - Wq.acnt[ac];
        f_try_anchor(Wq, e, Wq.outpos[lo + k], pi);
    }
    f_cta_sync();
}

/* select_matches (patterns.py:241-252): the stable sort key is (start_pos,
 * -len, list order), list order being pattern order then product order, which
 * for one pattern and one start is position order of the later members.  The
 * greedy scan keeps the smallest undecided key and drops what overlaps it.    */
template <class C> CLD unsigned long long f_key(const FW<C> &W, const FMatch &m) {
    const unsigned long long p1 = m.n > 1 ? W.posof[m.slot[1]] : 0xFFFFu, p2 = m.n > 2 ? W.posof[m.slot[2]] : 0xFFFFu;
    return (unsigned long long)W.posof[m.slot[0]] << 40 | (unsigned long long)(3u - m.n) << 38 | (unsigned long long)m.pat << 32 | p1 << 16 | p2;
}
template <class G, class C> CLF void f_select(const G &g, FW<C> &W) {
    const uint32_t nm = f_rd(g, &W.n_mt);
    uint32_t nsel = 0;
#pragma unroll 1
    for (;;) {
        unsigned long long best = NONE64;
        uint32_t bi = 0;
        FFOR(g, m, nm) if (m < nm && W.mstate[m] == MS_UNDECIDED) {
            const FMatch r = W.mt[m];
            bool clash = false;
#pragma unroll 1
            for (unsigned t = 0; t < r.n; t++) clash |= (W.sflag[r.slot[t]] & SF_TAKEN) != 0;
            if (clash) { W.mstate[m] = MS_REJECTED; continue; }
            const unsigned long long key = f_key(W, r);
            if (key < best) { best = key; bi = m; }
        }
        const unsigned long long win = g.min64(best);
        if (win == NONE64) break;
        if (best == win) {
            const FMatch r = W.mt[bi];
            W.mstate[bi] = MS_SELECTED;
            W.sel[nsel] = (uint16_t)bi;
#pragma unroll 1
            for (unsigned t = 0; t < r.n; t++) W.sflag[r.slot[t]] |= SF_TAKEN;
            a_add(&W.fstat[16 + r.pat], 1u);
        }
        nsel++;
        g.sync();
    }
    FFOR(g, j, nsel) if (j < nsel) { const FMatch r = W.mt[W.sel[j]]; for (unsigned t = 0; t < r.n; t++) W.sflag[r.slot[t]] &= (uint8_t)~SF_TAKEN; }
    if (g.rank == 0) W.n_sel = nsel;
    g.sync();
}

/* CL_EV_MATCH events of the round (emit_matches / MATCH_ONLY): positions are
 * block positions, idx carries the tuple's rank in itertools.product order    */
template <class G, class C> CLF void f_emit_matches(const G &g, FW<C> &W, const FEnv &e, uint32_t phase, cl_event *out, uint32_t cap) {
    const uint32_t nm = f_rd(g, &W.n_mt), nsel = f_rd(g, &W.n_sel), base = f_rd(g, &W.n_mev);
    if (g.rank == 0 && base + nm + nsel > cap) f_fail(W, F_REDO + 21);
    g.sync();
    if (!f_oks(g, W)) return;
    /* ccnt of every block that holds a match */
    FFOR(g, k, W.nb * MAX_CLS) if (k < W.nb * MAX_CLS) (&W.ccnt[0][0])[k] = 0;
    g.sync();
    {
        const uint16_t *o = W.ord[W.cur];
        FFOR(g, p, W.n_pos) if (p < W.n_pos) {
            const uint32_t s = o[p], fl = W.sflag[s];
            if ((fl & SF_LIVE) && (fl >> SF_CLS_SHIFT) != SF_NOCLS) a_add(&W.ccnt[W.sblk[s]][fl >> SF_CLS_SHIFT], 1u);
        }
    }
    g.sync();
    FFOR(g, m, nm) if (m < nm) {
        const FMatch r = W.mt[m];
        const FPat &p = e.P->p[r.pat];
        const uint32_t b = W.sblk[r.slot[0]], lo = W.bo[b];
        unsigned long long rank = 0;
#pragma unroll 1
        for (unsigned t = 0; t < r.n; t++) rank = (t ? rank * W.ccnt[b][p.t[t].cls] : 0ull) + f_class_rank(W, r.slot[t]);
        cl_event ev; ev.func = W.f; ev.seq = phase << 28 | b; ev.kind = CL_EV_MATCH; ev.idx = (uint32_t)r.pat << 20 | (uint32_t)rank;
        ev.a = r.pat; ev.b = W.posof[r.slot[0]] - lo; ev.c = r.n > 1 ? W.posof[r.slot[1]] - lo : NONE32; ev.d = r.n > 2 ? W.posof[r.slot[2]] - lo : NONE32;
        out[base + m] = ev;
    }
    /* selected matches: rank inside their block's select list */
    FFOR(g, j, nsel) if (j < nsel) {
        const FMatch r = W.mt[W.sel[j]];
        const uint32_t b = W.sblk[r.slot[0]], lo = W.bo[b];
        uint32_t jb = j;
        while (jb > 0 && W.sblk[W.mt[W.sel[jb - 1]].slot[0]] == b) jb--;
        cl_event ev; ev.func = W.f; ev.seq = phase << 28 | b; ev.kind = CL_EV_MATCH; ev.idx = 0x80000000u | (j - jb);
        ev.a = r.pat | 1u << 16; ev.b = W.posof[r.slot[0]] - lo; ev.c = r.n > 1 ? W.posof[r.slot[1]] - lo : NONE32; ev.d = r.n > 2 ? W.posof[r.slot[2]] - lo : NONE32;
        out[base + nm + j] = ev;
    }
    g.sync();
    if (g.rank == 0) W.n_mev = base + nm + nsel;
    g.sync();
}

/* ------------------------------------------------------------------ rewrites */
/* One lane runs the rewrites of a round in the reference's order.  Ids come
 * straight from the function's counters; new records go to the arena tail and
 * become part of the stream only when the rewrite succeeds (a refused rewrite
 * keeps the ids, values and immediates it allocated: G4).                    */
static constexpr uint16_t F_T_REL = 1u << 15;      /* slot payload is relative to the match's id bases (patched after the scan) */
/* what planning a match leaves for its commit (the plan itself is the chain of new records) */
struct FPlan { uint16_t head; uint8_t tq, nins, nv, ni, nq, flags; };      /* flags: rm (3 bits) | retag << 3 | ok << 4; tq: first staged immediate */
static_assert(sizeof(FPlan) == 8, "FPlan lives in the class-count table's storage");
template <class C> struct FRW {
    FW<C> *W; const FEnv *e;
    uint32_t s[3]; cl_hdr h[3];
    unsigned n, pat;
    uint32_t head, last, nins;     /* the plan's insert list: a chain of record slots (FW::nxt) */
    uint32_t nv, ni, nq;           /* values / instruction ids / immediates allocated so far, relative to the match */
    uint32_t tq_head, tq_last;     /* staged immediates (FW::timm), chained in creation order (FW::tnext) */
    uint32_t rm, retag, esc;       /* esc: bit 4t + k = def k of record t escapes (snapshot of the block's start) */
    uint32_t over;                 /* capacity of the slice exceeded: 1 values, 2 immediates, 4 def_iid log, 8 record slots */
};
/* a record slot: a freed one first, else the arena grows (any lane, any time between two frees) */
template <class C> CLD uint32_t f_alloc_slot(FW<C> &W) {
#if CL_DEV
    const int old = atomicSub((int *)&W.n_free, 1);
    if (old > 0) return W.fre[old - 1];
    atomicAdd((int *)&W.n_free, 1);
    const uint32_t s = atomicAdd(&W.n_slots, 1u);
    if (s < C::I) return s;
    atomicSub(&W.n_slots, 1u);
    return F_NONE;
#else
    if ((int)W.n_free > 0) return W.fre[--W.n_free];
    if (W.n_slots < C::I) return W.n_slots++;
    return F_NONE;
#endif
}
/* a removed record: its slot is free again, the values it defined have no defining record */
template <class C> CLD void f_free_slot(FW<C> &W, uint32_t s) {
    const uint32_t k = a_add(&W.n_free, 1u);
    if (k < C::I) W.fre[k] = (uint16_t)s;
}
template <class C> CLN void f_release(FW<C> &W, uint32_t s) {
    const cl_hdr h = W.hdr[s];
    f_value_defs(W, h, s, [&](uint32_t v) { if (v < C::V && W.defslot[v] == s) W.defslot[v] = F_NONE; });
    f_free_slot(W, s);
}
template <class C> CLD opnd frw_value(FRW<C> &c) {                 /* LiftedFunction.new_value("pair") */
    opnd o; o.tag = (uint16_t)(CL_K_VALUE | F_T_REL); o.pay = c.nv++;
    return o;
}
template <class C> CLD opnd frw_imm(FRW<C> &c, unsigned long long bits, unsigned long long text, bool hextext) {
    FW<C> &W = *c.W;
    const uint32_t t = c.nq < 255u ? a_add(&W.n_timm, 1u) : (uint32_t)C::TQ;
    opnd o; o.tag = (uint16_t)(CL_K_IMM | F_T_REL | (hextext ? CL_T_IMM_HEXTEXT : 0)); o.pay = c.nq | t << 8;      /* index in the match, staging slot */
    if (t < C::TQ) {
        W.timm[t].bits = bits; W.timm[t].text = text; W.tnext[t] = 0xFF;
        if (c.nq) W.tnext[c.tq_last] = (uint8_t)t; else c.tq_head = t;
        c.tq_last = t; c.nq++;
    } else c.over |= 2u;
    return o;
}
/* bits / spelling of an immediate operand, staged or already in the function's table */
template <class C> CLD cl_imm frw_imm_of(const FRW<C> &c, opnd o) {
    if (o.tag & F_T_REL) return c.W->timm[(o.pay >> 8) < C::TQ ? (o.pay >> 8) : 0];
    return f_imm_at(*c.W, *c.e, o.pay);
}
/* make_inst (ssir.py:237-241) + append to the plan's insert list; returns the (relative) iid.  The value the
 * record defines gets def_iid = this iid (patterns.py:297,309,356,384...): the log entry is written at commit */
template <class C> CLN uint32_t frw_emit(FRW<C> &c, uint16_t op, uint16_t modset, opnd def, const opnd *uses, unsigned nu) {
    FW<C> &W = *c.W;
    const uint32_t iid = c.ni++;
    const uint32_t s = f_alloc_slot(W);
    if (s == F_NONE) { c.over |= 8u; return iid; }
    cl_hdr h;
    h.iid = iid; h.op = op; h.modset = modset; h.n_defs = 1; h.n_aux = 0; h.n_uses = (uint8_t)nu; h.flags = 0; h.ext = 0;
    W.hdr[s] = h;
    uint16_t *tg = &W.tag[s * 8]; uint32_t *py = &W.pay[s * 8];
    tg[0] = def.tag; py[0] = def.pay;
#pragma unroll 1
    for (unsigned k = 0; k < 7; k++) { tg[1 + k] = k < nu ? uses[k].tag : (uint16_t)0; py[1 + k] = k < nu ? uses[k].pay : 0u; }
    W.sflag[s] = 0;
    W.nxt[s] = F_NONE;
    if (c.nins) W.nxt[c.last] = (uint16_t)s; else c.head = s;
    c.last = s; c.nins++;
    return iid;
}
template <class C> CLD void frw_drop(FRW<C> &c, opnd o) { if (is_value(o) && o.pay < C::V) c.W->alive[o.pay] = 0; }   /* _drop_values :314-317 */
/* _escapes (patterns.py:259-263) against the def-use snapshot of the block: a
 * value escapes iff it has more use sites than the group itself holds.  Evaluated
 * for every def of every selected match of a block before the block's first
 * rewrite (f_escape_bits), so the rewrites can update the use counts as they go. */
template <class C> CLN uint32_t f_escape_bits(const FW<C> &W, const FMatch &m) {
    FVals us[3];
#pragma unroll 1
    for (unsigned t = 0; t < 3; t++) { if (t < m.n) us[t] = f_uses(W, m.slot[t]); else us[t].n = 0; }
    uint32_t bits = 0;
#pragma unroll 1
    for (unsigned t = 0; t < m.n; t++) {
        const cl_hdr h = W.hdr[m.slot[t]];
        const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
#pragma unroll 1
        for (unsigned k = 0; k < nd && k < 4; k++) {
            const opnd d = f_slot(W, m.slot[t], d0 + k);
            if (!is_value(d) || d.pay >= C::V) continue;
            uint32_t inside = 0;
#pragma unroll 1
            for (unsigned u = 0; u < m.n; u++)
#pragma unroll 1
                for (uint32_t q = 0; q < us[u].n && q < 8; q++) inside += f_val(us[u], q) == d.pay;
            if (W.usecnt[d.pay] != inside) bits |= 1u << (4 * t + k);
        }
    }
    return bits;
}
template <class C> CLD bool frw_escapes(const FRW<C> &c, unsigned t, unsigned k) { return (c.esc >> (4 * t + k)) & 1u; }
/* _safe (patterns.py:266-275)                                                 */
template <class C> CLN bool frw_safe(FRW<C> &c, const opnd *redef, unsigned nredef) {
    FW<C> &W = *c.W;
#pragma unroll 1
    for (unsigned t = 0; t < c.n; t++) {
        const unsigned d0 = def0(c.h[t]), nd = (unsigned)c.h[t].n_defs + c.h[t].n_aux;
        if (nd > 4) { f_fail(W, F_REDO + 24); return false; }
#pragma unroll 1
        for (unsigned k = 0; k < nd; k++) {
            const opnd d = f_slot(W, c.s[t], d0 + k);
            if (!is_value(d)) continue;
            bool re = false;
#pragma unroll 1
            for (unsigned j = 0; j < nredef; j++) re |= is_value(redef[j]) && redef[j].pay == d.pay;
            if (!re && frw_escapes(c, t, k)) return false;
        }
    }
    return true;
}
/* _pack_pair (patterns.py:278-300); CL_K_NONE stands for None                 */
template <class C> CLN opnd frw_pack_pair(FRW<C> &c, opnd lo, opnd hi) {
    FW<C> &W = *c.W;
    const bool lo_zero = is_zero(lo), hi_zero = is_zero(hi);
    opnd none; none.tag = CL_K_NONE; none.pay = 0;
    if (lo_zero && hi_zero) return none;
    if (is_imm(lo) && hi_zero) {
        const cl_imm im = f_imm_at(W, *c.e, lo.pay);
        return frw_imm(c, im.bits & 0xFFFFFFFFull, im.text, (lo.tag & CL_T_IMM_HEXTEXT) != 0);
    }
    if (is_imm(lo) && is_imm(hi)) {
        const unsigned long long bits = (f_imm_at(W, *c.e, lo.pay).bits & 0xFFFFFFFFull) | (f_imm_at(W, *c.e, hi.pay).bits & 0xFFFFFFFFull) << 32;
        return frw_imm(c, bits, bits, true);
    }
    if (lo_zero && is_imm(hi)) {
        const unsigned long long bits = (f_imm_at(W, *c.e, hi.pay).bits & 0xFFFFFFFFull) << 32;
        return frw_imm(c, bits, bits, true);
    }
    const opnd d = frw_value(c);
    opnd u[2];
    u[0] = lo_zero ? frw_imm(c, 0, 0, true) : strip(lo);
    u[1] = hi_zero ? frw_imm(c, 0, 0, true) : strip(hi);
    const uint32_t iid = frw_emit(c, CL_OP_PACK64, CL_MS_NONE, d, u, 2);
    return d;
}
/* _unpack_into (patterns.py:303-311)                                          */
template <class C> CLN void frw_unpack_into(FRW<C> &c, opnd src, opnd lo_ref, opnd hi_ref) {
    FW<C> &W = *c.W;
    const opnd refs[2] = { lo_ref, hi_ref };
#pragma unroll 1
    for (int k = 0; k < 2; k++) {
        if (!is_value(refs[k])) continue;
        const opnd d = value_ref(refs[k].pay);
        const uint32_t iid = frw_emit(c, CL_OP_UNPACK64, k ? CL_MS_HI : CL_MS_LO, d, &src, 1);
        if (!(d.pay < C::V && W.alive[d.pay])) { f_fail(W, F_REDO + 5); return; }        /* KeyError */
        }
}
/* fn.values[res.vid].def_iid = agg.iid                                        */
template <class C> CLD bool frw_redefine(FRW<C> &c, opnd res, uint32_t iid) {
    FW<C> &W = *c.W;
    if (!is_value(res) || !(res.pay < C::V && W.alive[res.pay])) { f_fail(W, F_REDO + 6); return false; }   /* AttributeError / KeyError */
    (void)iid;
    return true;
}
template <class C> CLD opnd frw_use(const FRW<C> &c, unsigned t, unsigned k) { return f_slot(*c.W, c.s[t], use0(c.h[t]) + k); }
template <class C> CLD opnd frw_def(const FRW<C> &c, unsigned t, unsigned k) { return f_slot(*c.W, c.s[t], def0(c.h[t]) + k); }
template <class C> CLD opnd frw_aux(const FRW<C> &c, unsigned t, unsigned k) { return f_slot(*c.W, c.s[t], aux0(c.h[t]) + k); }

/* _rw_iadd364 (patterns.py:324-362)                                           */
template <class C> CLN bool frw_iadd364(FRW<C> &c) {
    const opnd carry = frw_aux(c, 0, 0);
    const opnd redef[2] = { frw_def(c, 0, 0), frw_def(c, 1, 0) };
    if (!frw_safe(c, redef, 2)) return false;
    opnd ops[3];
    unsigned nops = 0;
#pragma unroll 1
    for (unsigned k = 0; k < 3; k++) {
        const opnd lo_op = frw_use(c, 0, k), hi_op = frw_use(c, 1, k);
        const bool neg_lo = o_neg(lo_op), not_hi = o_not(hi_op);
        const bool plain = !neg_lo && !not_hi && !o_not(lo_op) && !o_neg(hi_op);
        if (plain) {
            const opnd p = frw_pack_pair(c, lo_op, hi_op);
            if (!is_none(p)) ops[nops++] = p;
        } else if (neg_lo && not_hi) {
            opnd p = frw_pack_pair(c, strip(lo_op), strip(hi_op));
            if (is_none(p)) return false;
            if (is_imm(p)) {                       /* Imm(-p.int_value(64) & M64, p.text) :348 */
                const cl_imm im = frw_imm_of(c, p);
                ops[nops++] = frw_imm(c, 0ull - im.bits, im.text, (p.tag & CL_T_IMM_HEXTEXT) != 0);
            } else {
                p.tag |= CL_T_NEG;
                ops[nops++] = p;
            }
        } else
            return false;                          /* mixed negation :353 */
    }
    if (!nops) return false;
    const opnd d = frw_value(c);
    const uint32_t iid = frw_emit(c, CL_OP_IADD364, CL_MS_NONE, d, ops, nops);
    frw_unpack_into(c, d, redef[0], redef[1]);
    frw_drop(c, carry);
    c.rm = 3;
    return true;
}
/* _rw_isetp64 (patterns.py:371-390)                                           */
template <class C> CLN bool frw_isetp64(FRW<C> &c) {
    const FProg &P = *c.e->P;
    const FPat &p = P.p[c.pat];
    const opnd res = frw_def(c, 1, 0);
    if (!frw_safe(c, &res, 1)) return false;
    const cl_modset &mlo = c.e->ms[c.h[0].modset];
    const unsigned cond = P.group_pos[mlo.first[p.cond_group & 3] & 63], bop = P.group_pos[mlo.first[p.bop_group & 3] & 63];
    const unsigned unsigned_hi = (c.e->ms[c.h[1].modset].mask >> CL_MB_U32) & 1u;
    opnd u[3];
    u[0] = frw_pack_pair(c, frw_use(c, 0, 0), frw_use(c, 1, 0));
    u[1] = frw_pack_pair(c, frw_use(c, 0, 1), frw_use(c, 1, 1));
    if (is_none(u[0])) u[0] = frw_imm(c, 0, 0, true);
    if (is_none(u[1])) u[1] = frw_imm(c, 0, 0, true);
    u[2] = frw_use(c, 1, 2);
    if (!is_value(res)) { f_fail(*c.W, F_REDO + 7); return false; }
    const uint32_t iid = frw_emit(c, CL_OP_ISETP64, P.isetp64_ms[cond & 7][unsigned_hi][bop & 7], value_ref(res.pay), u, 3);
    if (!frw_redefine(c, res, iid)) return false;
    frw_drop(c, frw_def(c, 0, 0));
    c.rm = 3;
    return true;
}
/* _rw_lea64 (patterns.py:393-411)                                             */
template <class C> CLN bool frw_lea64(FRW<C> &c) {
    const opnd carry = frw_aux(c, 0, 0);
    const opnd redef[2] = { frw_def(c, 0, 0), frw_def(c, 1, 0) };
    if (!frw_safe(c, redef, 2)) return false;
    const opnd a64 = frw_pack_pair(c, frw_use(c, 0, 0), frw_use(c, 1, 2));
    const opnd b64 = frw_pack_pair(c, frw_use(c, 0, 1), frw_use(c, 1, 1));
    if (is_none(a64) || is_none(b64)) return false;
    const opnd d = frw_value(c);
    const opnd u[3] = { b64, a64, frw_use(c, 0, 2) };
    const uint32_t iid = frw_emit(c, CL_OP_LEA64, CL_MS_NONE, d, u, 3);
    frw_unpack_into(c, d, redef[0], redef[1]);
    frw_drop(c, carry);
    c.rm = 3;
    return true;
}
/* tail of mov64 / cast64 / shl64 / shr64 (patterns.py:433-439 and alike): the
 * pack always goes, a feeder only when its result does not escape (G8)        */
template <class C> CLN bool frw_finish_pack(FRW<C> &c, unsigned n_feed) {
    c.rm = 1u << n_feed;
#pragma unroll 1
    for (unsigned t = 0; t < n_feed; t++) {
        const opnd d = frw_def(c, t, 0);
        if (!is_value(d)) { f_fail(*c.W, F_REDO + 8); return false; }
        if (!frw_escapes(c, t, 0)) { frw_drop(c, d); c.rm |= 1u << t; }
    }
    return true;
}
/* _rw_mov64 (patterns.py:421-439)                                             */
template <class C> CLN bool frw_mov64(FRW<C> &c) {
    const opnd clo = frw_use(c, 0, 0), chi = frw_use(c, 1, 0);
    if (kind_of(clo.tag) != CL_K_CONSTMEM || kind_of(chi.tag) != CL_K_CONSTMEM) return false;
    const uint32_t mask = (1u << CL_CM_OFFSET_BITS) - 1u;
    if ((clo.pay >> CL_CM_OFFSET_BITS) != (chi.pay >> CL_CM_OFFSET_BITS) || (chi.pay & mask) != (clo.pay & mask) + 4u) return false;
    const opnd res = frw_def(c, 2, 0);
    if (!is_value(res)) { f_fail(*c.W, F_REDO + 9); return false; }
    opnd u; u.tag = (uint16_t)(CL_K_CONSTMEM | 2u << CL_T_WIDTH_SHIFT); u.pay = clo.pay;
    const uint32_t iid = frw_emit(c, CL_OP_MOV64, CL_MS_NONE, value_ref(res.pay), &u, 1);
    if (!frw_redefine(c, res, iid)) return false;
    return frw_finish_pack(c, 2);
}
/* _rw_cast64 (patterns.py:442-453)                                            */
template <class C> CLN bool frw_cast64(FRW<C> &c) {
    const opnd res = frw_def(c, 1, 0);
    if (!is_value(res)) { f_fail(*c.W, F_REDO + 10); return false; }
    const opnd u = strip(frw_use(c, 1, 0));
    const uint32_t iid = frw_emit(c, CL_OP_CAST64, CL_MS_NONE, value_ref(res.pay), &u, 1);
    if (!frw_redefine(c, res, iid)) return false;
    return frw_finish_pack(c, 1);
}
/* _rw_shl64 / _rw_shr64 (patterns.py:456-495)                                 */
template <class C> CLN bool frw_shift64(FRW<C> &c, bool right) {
    const bool is_signed = (c.e->ms[c.h[0].modset].mask >> CL_MB_S32) & 1u;
    const opnd src = right ? frw_pack_pair(c, frw_use(c, 1, 0), frw_use(c, 0, 2)) : frw_pack_pair(c, frw_use(c, 0, 0), frw_use(c, 0, 2));
    if (is_none(src)) return false;
    const opnd res = frw_def(c, 2, 0);
    if (!is_value(res)) { f_fail(*c.W, F_REDO + 11); return false; }
    const opnd u[2] = { src, frw_use(c, 0, 1) };
    const uint32_t iid = frw_emit(c, right ? CL_OP_SHR64 : CL_OP_SHL64, right ? (is_signed ? CL_MS_S64 : CL_MS_U64) : CL_MS_NONE, value_ref(res.pay), u, 2);
    if (!frw_redefine(c, res, iid)) return false;
    return frw_finish_pack(c, 2);
}
/* Binding of a pattern variable = key of the first slot that mentions it, then
 * _var_operand (patterns.py:514-524)                                          */
template <class C> CLN bool frw_var_operand(FRW<C> &c, unsigned which, opnd *out) {
    const FPat &p = c.e->P->p[c.pat];
    const unsigned t = p.var_t[which], k = p.var_k[which];
    if (t >= c.n) { f_fail(*c.W, F_REDO + 12); return false; }
    const opnd o = f_slot(*c.W, c.s[t], has_guard(c.h[t]) + k);
    switch (kind_of(o.tag)) {
    case CL_K_VALUE: *out = value_ref(o.pay); return true;
    case CL_K_IMM: { const unsigned long long b = f_imm_at(*c.W, *c.e, o.pay).bits; *out = frw_imm(c, b, b, true); return true; }
    case CL_K_CONSTMEM: out->tag = (uint16_t)(CL_K_CONSTMEM | 1u << CL_T_WIDTH_SHIFT); out->pay = o.pay; return true;
    case CL_K_RZ: case CL_K_URZ: out->tag = CL_K_RZ; out->pay = 0; return true;
    default: f_fail(*c.W, F_REDO + 13); return false;                                  /* AssertionError */
    }
}
/* _rw_xmad (patterns.py:498-511)                                              */
template <class C> CLN bool frw_xmad(FRW<C> &c) {
    const opnd dres = frw_def(c, 2, 0);
    if (!frw_safe(c, &dres, 1)) return false;
    opnd u[3];
    if (!frw_var_operand(c, 0, &u[0])) return false;
    if (!frw_var_operand(c, 1, &u[1])) return false;
    if (!frw_var_operand(c, 2, &u[2])) return false;
    if (!is_value(dres)) { f_fail(*c.W, F_REDO + 14); return false; }
    const uint32_t iid = frw_emit(c, CL_OP_IMAD, CL_MS_NONE, value_ref(dres.pay), u, 3);
    if (!frw_redefine(c, dres, iid)) return false;
#pragma unroll 1
    for (unsigned t = 0; t < 2; t++)
#pragma unroll 1
        for (unsigned k = 0; k < c.h[t].n_defs; k++) frw_drop(c, frw_def(c, t, k));
    c.rm = 7;
    return true;
}
template <class C> CLN bool frw_run(FRW<C> &c) {
    switch (c.e->P->p[c.pat].rewrite) {
    case CL_RW_IADD364: return frw_iadd364(c);
    case CL_RW_ISETP64: return frw_isetp64(c);
    case CL_RW_LEA64: return frw_lea64(c);
    case CL_RW_IMAD_WIDE: c.retag = 1; return true;             /* _rw_imad_wide :414-418 */
    case CL_RW_MOV64: return frw_mov64(c);
    case CL_RW_CAST64: return frw_cast64(c);
    case CL_RW_SHL64: return frw_shift64(c, false);
    case CL_RW_SHR64: return frw_shift64(c, true);
    case CL_RW_XMAD: return frw_xmad(c);
    }
    f_fail(*c.W, F_REDO + 15);
    return false;
}

/* The plan of one selected match becomes part of the function, or is refused:
 * the ids it allocated relative to the match get their bases (exclusive scan
 * over the matches of the batch in select order = the reference's allocation
 * order, G3; a refused plan keeps its ids, values and immediates, G4).  The use
 * counts follow the edit at once; the escape tests of the block's other matches
 * were taken before (at planning), which is the reference's per-block def-use
 * snapshot (patterns.py:674,706).  Runs on many lanes at once, one match each. */
template <class C> CLF void f_commit(FW<C> &W, const FEnv &e, unsigned table, uint32_t phase, const FMatch m, const FPlan pl,
                                     uint32_t vbase, uint32_t ibase, uint32_t qbase, uint32_t lbase, uint32_t rank_in_block) {
    const FProg &P = *e.P;
    const uint32_t b = W.sblk[m.slot[0]];
    const bool ok = (pl.flags >> 4) & 1u;
#pragma unroll 1
    for (uint32_t k = 0; k < pl.nv; k++) {
        const uint32_t v = vbase + k;
        W.alive[v] = 1; W.usecnt[v] = 0; W.defslot[v] = F_NONE; W.norigin[v] = 1u << 14;
    }
    {
        uint32_t t = pl.tq;
#pragma unroll 1
        for (uint32_t k = 0; k < pl.nq; k++) { W.newimm[qbase - W.nq_in + k] = W.timm[t]; t = W.tnext[t]; }
    }
    {
        uint32_t s = pl.head;
#pragma unroll 1
        for (uint32_t r = 0; r < pl.nins; r++, s = W.nxt[s]) {
            const uint32_t iid = W.hdr[s].iid + ibase, ns = 1u + W.hdr[s].n_uses;
            W.hdr[s].iid = iid;
#pragma unroll 1
            for (uint32_t k = 0; k < ns; k++) {
                const uint16_t t = W.tag[s * 8 + k];
                if (!(t & F_T_REL)) continue;
                W.pay[s * 8 + k] = kind_of(t) == CL_K_VALUE ? W.pay[s * 8 + k] + vbase : (W.pay[s * 8 + k] & 0xFFu) + qbase;
                W.tag[s * 8 + k] = (uint16_t)(t & ~F_T_REL);
            }
            W.dlog[lbase + r].vid = W.pay[s * 8]; W.dlog[lbase + r].iid = (int32_t)iid;     /* value.def_iid = inst.iid */
        }
    }
    if (!ok) {
        uint32_t s = pl.head;
#pragma unroll 1
        for (uint32_t r = 0; r < pl.nins; r++) { const uint32_t nx = W.nxt[s]; f_free_slot(W, s); s = nx; }      /* the plan is dropped, its ids are not (G4) */
        a_add(&W.fstat[48 + m.pat], 1u);
        f_event(W, phase << 28 | b, CL_EV_REFUSED, rank_in_block, m.pat, W.blk[b].bid, 0, 0);
        return;
    }
    /* removed records first (their values lose their defining record) */
#pragma unroll 1
    for (unsigned t = 0; t < m.n; t++) if (pl.flags >> t & 1u) {
        const uint32_t s = m.slot[t];
        W.sflag[s] = 0;
        f_value_operands(W, W.hdr[s], s, [&](uint32_t v) { f_dec_use(W, v); });
        f_release(W, s);
    }
    const uint32_t anchor = m.slot[m.n - 1], ap = W.posof[anchor];
    {
        uint32_t s = pl.head;
#pragma unroll 1
        for (uint32_t r = 0; r < pl.nins; r++, s = W.nxt[s]) {
            const cl_hdr h = W.hdr[s];
            unsigned sf = SF_LIVE | SF_INS | f_cls(P, table, h.op) << SF_CLS_SHIFT;
            if (h.op < CL_OP__COUNT && (P.opflags[h.op] & CL_OPF_PURE)) sf |= SF_PURE;
            W.sflag[s] = (uint8_t)sf;
            W.sblk[s] = (uint8_t)b;
            W.posof[s] = (uint16_t)ap;
            const opnd d = f_slot(W, s, 0);
            if (is_value(d) && d.pay < C::V) W.defslot[d.pay] = (uint16_t)s;
            f_value_operands(W, h, s, [&](uint32_t v) { f_inc_use(W, v); });
        }
    }
    if (pl.nins) { W.insslot[ap] = pl.head; W.inscnt[ap] = 1; }
    if (pl.flags & 8u) {                            /* _rw_imad_wide :414-418 */
        cl_hdr &h = W.hdr[m.slot[0]];
        h.modset = e.ms[h.modset].minus_wide;
        h.op = CL_OP_IMAD64;
        W.sflag[m.slot[0]] = (uint8_t)((W.sflag[m.slot[0]] & 15u) | f_cls(P, table, CL_OP_IMAD64) << SF_CLS_SHIFT);
    }
    if (pl.nins || (pl.flags & 7u)) W.dirty = 1;
    a_add(&W.fstat[32 + m.pat], 1u);
}

/* _apply_patterns (patterns.py:671-707), the rewrite half, in steps the CTA takes
 * together.  A step is one block of every resident function (blocks in order:
 * the escape tests of a block see the use counts the earlier blocks left, G5):
 *   f_plan_prep    group: the block's selected matches [j0, j1), sorted by pattern
 *   f_plan_pooled  CTA: one lane plans one match (any function's), full warps per pattern
 *   f_plan_commit  group: id bases by scan in select order, then the edits          */
template <class C> CLD FPlan *f_plans(FW<C> &W) { return (FPlan *)&W.ccnt[0][0]; }
template <class G, class C> CLF void f_plan_prep(const G &g, FW<C> &W, const FCtx<C> &x, bool on) {
    FFOR(g, k, 2 * CL_MAX_PATTERNS) if (k < 2 * CL_MAX_PATTERNS) W.acnt[k] = 0;
    if (g.rank == 0) W.n_timm = 0;
    g.sync();
    const uint32_t nsel = on ? W.n_sel : 0u;
    /* counting sort of the selected matches by pattern: acnt[pi] counts, acnt[16 + pi] fill cursors, psel = indices j */
    uint16_t *psel = W.esc;
    FFOR(g, j, nsel) if (j < nsel) a_add(&W.acnt[W.mt[W.sel[j]].pat & 15u], 1u);
    g.sync();
    if (g.rank == 0) {
        uint32_t run = 0;
#pragma unroll 1
        for (unsigned pi = 0; pi < CL_MAX_PATTERNS; pi++) { W.acnt[CL_MAX_PATTERNS + pi] = run; run += W.acnt[pi]; }
    }
    g.sync();
    FFOR(g, j, nsel) if (j < nsel) psel[a_add(&W.acnt[CL_MAX_PATTERNS + (W.mt[W.sel[j]].pat & 15u)], 1u)] = (uint16_t)j;
    FFOR(g, pi, CL_MAX_PATTERNS) if (pi < CL_MAX_PATTERNS) x.Q->cnt[x.gi][pi] = W.acnt[pi];
    g.sync();
}
template <class C> CLF void f_plan_pooled(const FCtx<C> &x, const FEnv &e) {
    const uint32_t total = f_pool_layout(x);
#pragma unroll 1
    for (uint32_t i = x.tid; i < total; i += x.nthreads) {
        uint32_t pi, gq, k;
        f_pool_item(x, i, pi, gq, k);
        FW<C> &W = x.w(gq);
        const uint32_t j = W.esc[W.acnt[CL_MAX_PATTERNS + pi] - W.acnt[pi] + k];
        const FMatch m = W.mt[W.sel[j]];
        FRW<C> c;
        c.W = &W; c.e = &e; c.n = m.n; c.pat = m.pat; c.head = F_NONE; c.last = F_NONE; c.nins = 0; c.nv = 0; c.ni = 0; c.nq = 0;
        c.tq_head = 0xFF; c.tq_last = 0xFF; c.rm = 0; c.retag = 0; c.over = 0;
        c.esc = f_escape_bits(W, m);
#pragma unroll 1
        for (unsigned t = 0; t < 3; t++) { c.s[t] = t < m.n ? m.slot[t] : (uint32_t)m.slot[0]; c.h[t] = W.hdr[c.s[t]]; }
        const bool ok = frw_run(c);
        if (c.over || c.nins > 255u || c.nv > 255u || c.ni > 255u) f_fail(W, F_REDO + 40 + (c.over ? c.over : 8u));
        if (ok && c.rm && W.nb > 1) {
            /* G5: every block is planned against the use counts of the round's start; the reference lets a block see
             * the rewrites of the blocks before it.  That differs only when a removed record uses a value defined in
             * a LATER block of its function (then a later escape test would count one use less): hand back.          */
            const uint32_t b = W.sblk[m.slot[0]];
#pragma unroll 1
            for (unsigned t = 0; t < m.n; t++) if (c.rm >> t & 1u)
                f_value_operands(W, c.h[t], m.slot[t], [&](uint32_t v) {
                    const uint32_t dp = v < C::V ? W.defslot[v] : (uint32_t)F_NONE;
                    if (dp != F_NONE && W.sblk[dp] > b) f_fail(W, F_REDO + 25);
                });
        }
        FPlan pl;
        pl.head = (uint16_t)c.head; pl.tq = (uint8_t)c.tq_head; pl.nins = (uint8_t)c.nins; pl.nv = (uint8_t)c.nv; pl.ni = (uint8_t)c.ni; pl.nq = (uint8_t)c.nq;
        pl.flags = (uint8_t)((c.rm & 7u) | (c.retag ? 8u : 0u) | (ok ? 16u : 0u));
        f_plans(W)[j] = pl;
    }
    f_cta_sync();
}
/* returns the number of successful rewrites of the step */
template <class G, class C> CLF uint32_t f_plan_commit(const G &g, FW<C> &W, const FEnv &e, unsigned table, uint32_t phase) {
    const uint32_t nsel = f_rd(g, &W.n_sel);
    uint32_t done = 0;
    if (!f_oks(g, W)) return 0;
#pragma unroll 1
    for (uint32_t c0 = 0; c0 < nsel; c0 += g.size) {
        g.sync();
        const uint32_t nv0 = W.next_vid, ni0 = W.next_iid, nq0 = W.nq_in + W.n_newimm, nl0 = W.n_log;
        const uint32_t j = c0 + g.rank;
        const bool act = j < nsel;
        FPlan pl; pl.head = F_NONE; pl.tq = 0xFF; pl.nins = pl.nv = pl.ni = pl.nq = pl.flags = 0;
        FMatch m; m.n = 0; m.pat = 0; m.slot[0] = m.slot[1] = m.slot[2] = 0;
        uint32_t rank_in_block = 0;
        if (act) {
            pl = f_plans(W)[j];
            m = W.mt[W.sel[j]];
            /* rank of the match inside its block's select list (diagnostics, patterns.py:684) */
            const uint32_t b = W.sblk[m.slot[0]];
            uint32_t jb = j;
#pragma unroll 1
            while (jb > 0 && W.sblk[W.mt[W.sel[jb - 1]].slot[0]] == b) jb--;
            rank_in_block = j - jb;
        }
        /* id bases: two packed scans (11 bits per count: at most 8 of each per match, 128 lanes) */
        uint32_t t1, t2;
        const uint32_t x1 = g.exscan((uint32_t)pl.nv | (uint32_t)pl.ni << 11 | (uint32_t)pl.nq << 22, t1), x2 = g.exscan((uint32_t)pl.nins | ((pl.flags >> 4) & 1u) << 11, t2);
        const uint32_t vb = x1 & 0x7FFu, ib = (x1 >> 11) & 0x7FFu, qb = x1 >> 22, lb = x2 & 0x7FFu;
        const uint32_t tv = t1 & 0x7FFu, ti = (t1 >> 11) & 0x7FFu, tq = t1 >> 22, tl = t2 & 0x7FFu, tok = t2 >> 11;
        if (g.rank == 0 && (nv0 + tv > C::V || nq0 - W.nq_in + tq > C::Q || nl0 + tl > C::L)) f_fail(W, F_REDO + 45);
        g.sync();
        if (!f_oks(g, W)) return done;
        if (act) f_commit(W, e, table, phase, m, pl, nv0 + vb, ni0 + ib, nq0 + qb, nl0 + lb, rank_in_block);
        g.sync();
        if (g.rank == 0) { W.next_vid = nv0 + tv; W.next_iid = ni0 + ti; W.n_newimm = nq0 - W.nq_in + tq; W.n_log = nl0 + tl; }
        done += tok;
        /* a new pure record nobody reads is dead on arrival */
        if (act && (pl.flags & 16u)) {
            uint32_t s = pl.head;
#pragma unroll 1
            for (uint32_t r = 0; r < pl.nins; r++, s = W.nxt[s]) {
                if (!(W.sflag[s] & SF_PURE)) continue;
                const opnd d = f_slot(W, s, 0);
                if (is_value(d) && d.pay < C::V && W.usecnt[d.pay] == 0) f_push_wl(W, s);
            }
        }
        g.sync();
    }
    return done;
}

/* ------------------------------------------------------- dead pseudo ops */
/* remove_dead_pseudo (patterns.py:771-791).  The reference removes, round by
 * round, every pure instruction whose values have no users: the least fixpoint
 * of "dead", reached here by chaotic iteration.  The first call looks at every
 * record; afterwards a record can only die when one of its values loses its
 * last user (or when it is inserted unused), and those are on the worklist.   */
template <class C> CLN void f_try_kill(FW<C> &W, uint32_t s) {
    const uint32_t fl = W.sflag[s];
    if ((fl & (SF_LIVE | SF_PURE)) != (SF_LIVE | SF_PURE)) return;
    const cl_hdr h = W.hdr[s];
    unsigned nd = 0; bool used = false;
    f_value_defs(W, h, s, [&](uint32_t v) { nd++; used |= v < C::V && *(volatile uint32_t *)&W.usecnt[v] != 0; });
    if (!nd || used) return;
#if CL_DEV
    {   /* claim the record: two lanes may hold it (worklist duplicates) */
        uint32_t *w = (uint32_t *)&W.sflag[s & ~3u];
        const uint32_t bit = (uint32_t)SF_LIVE << (8u * (s & 3u));
        if (!(atomicAnd(w, ~bit) & bit)) return;
    }
#else
    W.sflag[s] = (uint8_t)(fl & ~SF_LIVE);
#endif
    f_value_defs(W, h, s, [&](uint32_t v) { if (v < C::V) W.alive[v] = 0; });
    f_value_operands(W, h, s, [&](uint32_t v) { f_dec_use(W, v); });
    f_release(W, s);
    W.dirty = 1;
}
template <class G, class C> CLF void f_dce(const G &g, FW<C> &W) {
    g.sync();
    uint32_t head = 0;
    bool sweep = !(f_rd(g, &W.flags) & FF_SWEPT);
#pragma unroll 1
    for (;;) {
        const uint32_t fl = f_rd(g, &W.flags), tl = f_rd(g, &W.wl_tail);
        if (sweep || (fl & FF_WLOVER)) {            /* first call, or the worklist lost entries: look at every record */
            if (g.rank == 0) { W.flags = (fl | FF_SWEPT) & ~(uint32_t)FF_WLOVER; W.wl_tail = 0; }
            g.sync();
            const uint32_t n = W.n_slots;
            FFOR(g, s, n) if (s < n) f_try_kill(W, s);
            g.sync();
            head = 0; sweep = false;
            continue;
        }
        const uint32_t tail = tl < C::I ? tl : C::I;
        if (head >= tail) break;
        FFOR(g, k, tail - head) if (k < tail - head) f_try_kill(W, W.wl[head + k]);
        head = tail;
        g.sync();
    }
    if (g.rank == 0) W.wl_tail = 0;
    g.sync();
}

/* ------------------------------------------------------------ pack folding */
/* simplify_packs + _redirect_values (patterns.py:710-764); returns `changed` */
template <class C> CLD uint32_t f_final_of(const FW<C> &W, uint32_t v) {
    while (v < C::V && W.redirect[v] != F_NONE) v = W.redirect[v];
    return v;
}
template <class G, class C> CLF uint32_t f_simplify(const G &g, FW<C> &W, const FEnv &e) {
    if (g.rank == 0) W.nred = 0;
    g.sync();
    const uint32_t n = W.n_slots;
    uint16_t *cand = W.outpos;                     /* (d, s) pairs; free between rebuilds */
    FFOR(g, s, n) if (s < n) {
        if (!f_live(W, s)) continue;
        const cl_hdr h = W.hdr[s];
        if (h.op != CL_OP_PACK64 || h.n_uses != 2) continue;
        const unsigned u0 = use0(h);
        const opnd lo = f_slot(W, s, u0), hi = f_slot(W, s, u0 + 1);
        if (!is_value(lo) || !is_value(hi)) continue;
        if ((lo.tag | hi.tag) & (CL_T_NEG | CL_T_NOT)) continue;
        if (lo.pay >= C::V || hi.pay >= C::V) continue;
        const uint32_t plo = W.defslot[lo.pay], phi = W.defslot[hi.pay];
        if (plo == F_NONE || phi == F_NONE || !f_live(W, plo) || !f_live(W, phi)) continue;
        const cl_hdr dlo = W.hdr[plo], dhi = W.hdr[phi];
        if (dlo.op != CL_OP_UNPACK64 || dhi.op != CL_OP_UNPACK64) continue;
        if (!((e.ms[dlo.modset].mask >> CL_MB_LO) & 1u) || !((e.ms[dhi.modset].mask >> CL_MB_HI) & 1u)) continue;
        if (!dlo.n_uses || !dhi.n_uses) { f_fail(W, F_REDO + 17); continue; }       /* IndexError */
        const opnd slo = f_slot(W, plo, use0(dlo)), shi = f_slot(W, phi, use0(dhi));
        if (!(is_value(slo) && is_value(shi) && slo.pay == shi.pay)) continue;
        if (!h.n_defs) { f_fail(W, F_REDO + 18); continue; }
        const opnd d = f_slot(W, s, def0(h));
        if (!is_value(d) || d.pay >= C::V) { f_fail(W, F_REDO + 19); continue; }
        const uint32_t k = a_add(&W.nred, 1u);
        if (2 * k + 1 < C::I) { cand[2 * k] = (uint16_t)d.pay; cand[2 * k + 1] = (uint16_t)slo.pay; }
    }
    g.sync();
    const uint32_t changed = f_rd(g, &W.nred);
    if (!f_oks(g, W) || !changed) return changed;
    const uint32_t nv = W.next_vid;
    FFOR(g, v, nv) if (v < nv) W.redirect[v] = F_NONE;
    g.sync();
    FFOR(g, k, changed) if (k < changed) W.redirect[cand[2 * k]] = cand[2 * k + 1];
    g.sync();
    /* the use counts follow the redirects (every use site of the old value becomes one of the new) */
    auto move_use = [&](uint32_t v) {
        if (v >= C::V || W.redirect[v] == F_NONE) return;
        const uint32_t fo = f_final_of(W, v);
        f_inc_use(W, fo);
        f_dec_use(W, v);
    };
    FFOR(g, s, n) if (s < n && f_live(W, s)) f_value_operands(W, W.hdr[s], s, move_use);
    FFOR(g, b, W.nb) if (b < W.nb)
#pragma unroll 1
        for (int k = 0; k < 2; k++) if (kind_of(W.blk[b].term_tag[k]) == CL_K_VALUE) move_use(W.blk[b].term_pay[k]);
    g.sync();
    FFOR(g, s, n) if (s < n && f_live(W, s)) {
        const cl_hdr h = W.hdr[s];
        const unsigned u0 = use0(h);
#pragma unroll 1
        for (unsigned k = 0; k < h.n_uses; k++) {
            const opnd u = f_slot(W, s, u0 + k);
            if (is_value(u)) { if (u.pay < C::V && W.redirect[u.pay] != F_NONE) W.pay[s * 8 + u0 + k] = f_final_of(W, u.pay); }
            else if (kind_of(u.tag) == CL_K_MEMREF && u.pay < C::MR) {
                cl_memref &m = W.mem[u.pay];
                if (kind_of(m.base_tag) == CL_K_VALUE) m.base_pay = f_final_of(W, m.base_pay);
                if (kind_of(m.ureg_tag) == CL_K_VALUE) m.ureg_pay = f_final_of(W, m.ureg_pay);
            }
        }
        if (has_guard(h)) { const opnd gd = f_slot(W, s, 0); if (is_value(gd)) W.pay[s * 8] = f_final_of(W, gd.pay); }
    }
    FFOR(g, b, W.nb) if (b < W.nb)
#pragma unroll 1
        for (int k = 0; k < 2; k++) if (kind_of(W.blk[b].term_tag[k]) == CL_K_VALUE) W.blk[b].term_pay[k] = f_final_of(W, W.blk[b].term_pay[k]);
    g.sync();
    f_dce(g, W);
    return changed;
}

/* tag_cuda_objects (patterns.py:895-916)                                      */
template <class G, class C> CLF void f_tag(const G &g, FW<C> &W, const FEnv &e) {
    const uint32_t n = W.n_slots;
    FFOR(g, s, n) if (s < n && f_live(W, s)) {
        cl_hdr h = W.hdr[s];
        if (h.op != CL_OP_BAR && h.op != CL_OP_WARPSYNC && h.op != CL_OP_SHFL) continue;
        unsigned kind = 0, use = 7;
        const unsigned u0 = use0(h);
        if (h.op == CL_OP_BAR) {
            if ((e.ms[h.modset].mask >> CL_MB_SYNC) & 1u) {
                kind = 1;
#pragma unroll 1
                for (unsigned k = 0; k < h.n_uses && k < 7; k++) if (is_imm(f_slot(W, s, u0 + k))) use = k;
            }
        } else if (h.op == CL_OP_WARPSYNC) {
#pragma unroll 1
            for (unsigned k = 0; k < h.n_uses && k < 7; k++) {
                const opnd u = f_slot(W, s, u0 + k);
                if (is_imm(u)) { if (f_imm_at(W, e, u.pay).bits == 0xFFFFFFFFull) { kind = 2; use = k; } break; }
            }
        } else
            kind = 3;
        if (kind) {
            h.flags &= (uint8_t)~(CL_IF_OBJ_MASK | CL_IF_OBJUSE_MASK);
            h.flags |= (uint8_t)(kind << CL_IF_OBJ_SHIFT | use << CL_IF_OBJUSE_SHIFT);
            W.hdr[s].flags = h.flags;
        }
    }
    g.sync();
}

/* ------------------------------------------------------- reciprocal chains */
/* normalize_reciprocal (patterns.py:817-888), chains in parallel.
 *   R_k(r): an F2I is reachable from record r in <= k def-use hops (_reaches_f2i :850)
 *           -- backward propagation from the F2I records, three sweeps;
 *   a chain (MUFU.RCP of an I2F, IADD/IADD3 with an immediate using it) is accepted iff R_3(add);
 *   its number (vids, iids, boundary index) is its rank by (mufu, add) position.
 * The reference rewrites chain after chain on a rebuilt def-use graph; a later chain
 * sees an earlier one only if its search walks over that chain's add or MUFU.
 * Functions where an accepted add reaches the add or MUFU of an earlier chain
 * within two hops, adds with two reciprocal operands and every exception path of
 * the reference are handed back to the sequential kernel.                      */
enum { FRF_R0 = 1, FRF_R1 = 2, FRF_R2 = 4, FRF_R3 = 8, FRF_SEED = 16, FRF_MUFU = 128 };
struct FChain { uint16_t add, mufu, rcp, addv; };
static_assert(sizeof(FChain) == sizeof(FMatch), "chains live in the match list's storage");

template <class G, class C> CLF void f_reciprocal(const G &g, FW<C> &W, const FEnv &e) {
    const uint32_t n = W.n_slots, nv = W.next_vid;
    uint8_t *rflag = (uint8_t *)W.outpos;           /* [I]  per slot                    */
    uint8_t *valbits = (uint8_t *)W.redirect;       /* [V]  per value (propagation)     */
    FChain *chain = (FChain *)W.mt;                 /* [M]                              */
    uint8_t *crank = W.mstate;                      /* [M]  rank of the chain           */
    FFOR(g, v, nv) if (v < nv) valbits[v] = 0;
    if (g.rank == 0) W.n_mt = 0;
    /* R_0 and the MUFU.RCP records fed by an I2F */
    FFOR(g, s, n) if (s < n) {
        uint8_t fl = 0;
        if (f_live(W, s)) {
            const cl_hdr h = W.hdr[s];
            if (h.op == CL_OP_F2I) fl = (uint8_t)(FRF_R0 | FRF_R1 | FRF_R2 | FRF_R3);
            else if (h.op == CL_OP_MUFU && ((e.ms[h.modset].mask >> CL_MB_RCP) & 1u) && h.n_uses) {
                const opnd src = f_slot(W, s, use0(h));
                if (is_value(src) && src.pay < C::V) {
                    const uint32_t dp = W.defslot[src.pay];
                    if (dp != F_NONE && f_live(W, dp) && W.hdr[dp].op == CL_OP_I2F) {
                        if (!h.n_defs || !is_value(f_slot(W, s, def0(h)))) f_fail(W, F_REDO + 30);     /* IndexError / AttributeError */
                        else fl |= FRF_MUFU;
                    }
                }
            }
        }
        rflag[s] = fl;
    }
    g.sync();
#pragma unroll 1
    for (unsigned k = 1; k <= 3; k++) {
        const uint8_t prev = (uint8_t)(1u << (k - 1)), cur = (uint8_t)(1u << k);
        FFOR(g, s, n) if (s < n && (rflag[s] & prev)) f_value_operands(W, W.hdr[s], s, [&](uint32_t v) { if (v < C::V) valbits[v] |= cur; });
        g.sync();
        FFOR(g, s, n) if (s < n && f_live(W, s) && !(rflag[s] & cur)) {
            bool r = false;
            f_value_defs(W, W.hdr[s], s, [&](uint32_t v) { r |= v < C::V && (valbits[v] & cur); });
            if (r) rflag[s] |= (uint8_t)((0xFu << k) & 0xFu);        /* R_k implies R_k+1.. */
        }
        g.sync();
    }
    /* accepted chains */
    FFOR(g, s, n) if (s < n && f_live(W, s)) {
        const cl_hdr h = W.hdr[s];
        if (h.op != CL_OP_IADD && h.op != CL_OP_IADD3) continue;
        bool any_imm = false;
        const unsigned u0 = use0(h);
#pragma unroll 1
        for (unsigned k = 0; k < h.n_uses; k++) any_imm |= is_imm(f_slot(W, s, u0 + k));
        if (!any_imm) continue;
        unsigned hits = 0;
        uint32_t mp = F_NONE, rcp = 0;
        f_value_operands(W, h, s, [&](uint32_t v) {
            const uint32_t dp = v < C::V ? W.defslot[v] : (uint32_t)F_NONE;
            if (dp == F_NONE || !(rflag[dp] & FRF_MUFU)) return;
            const opnd d0 = f_slot(W, dp, def0(W.hdr[dp]));
            if (!is_value(d0) || d0.pay != v) return;
            hits++; mp = dp; rcp = v;
        });
        if (!hits) continue;
        if (hits > 1 || has_guard(h)) { f_fail(W, F_REDO + 31); continue; }
        if (!(rflag[s] & FRF_R3)) continue;
        if (W.sblk[mp] != W.sblk[s] || !h.n_defs || !is_value(f_slot(W, s, def0(h)))) { f_fail(W, F_REDO + 32); continue; }   /* KeyError :886 and friends */
        const uint32_t c = a_add(&W.n_mt, 1u);
        if (c < C::M) { FChain ch; ch.add = (uint16_t)s; ch.mufu = (uint16_t)mp; ch.rcp = (uint16_t)rcp; ch.addv = (uint16_t)f_slot(W, s, def0(h)).pay; chain[c] = ch; }
        else f_fail(W, F_REDO + 33);
    }
    g.sync();
    const uint32_t nc = f_rd(g, &W.n_mt);
    if (!f_oks(g, W) || nc == 0) return;
    if (nc > 127) { if (g.rank == 0) f_fail(W, F_REDO + 34); g.sync(); return; }
    /* order of the chains = the reference's processing order */
    FFOR(g, c, nc) if (c < nc) {
        const uint32_t key = (uint32_t)W.posof[chain[c].mufu] << 16 | W.posof[chain[c].add];
        uint32_t r = 0;
#pragma unroll 1
        for (uint32_t o = 0; o < nc; o++) r += ((uint32_t)W.posof[chain[o].mufu] << 16 | W.posof[chain[o].add]) < key;
        crank[c] = (uint8_t)r;
    }
    /* interference */
    uint16_t *own = W.insslot, *rch = W.wl;          /* per slot: own seed order, smallest order reached in one hop */
    uint16_t *vch = W.vtmp;                          /* per value: chain whose add defines it                       */
    uint32_t *qmin = &W.ccnt[0][0];                  /* per chain: smallest order reached in two hops                */
    FFOR(g, s, n) if (s < n) { own[s] = F_NONE; rch[s] = F_NONE; }
    FFOR(g, v, nv) if (v < nv) vch[v] = F_NONE;
    FFOR(g, c, nc) if (c < nc) qmin[c] = NONE32;
    g.sync();
    FFOR(g, c, nc) if (c < nc) {
        const FChain ch = chain[c];
        own[ch.add] = crank[c];
        bool first = true;                           /* the earliest chain of a MUFU names it */
#pragma unroll 1
        for (uint32_t o = 0; o < nc; o++) first &= !(chain[o].mufu == ch.mufu && crank[o] < crank[c]);
        if (first) own[ch.mufu] = crank[c];
        f_value_defs(W, W.hdr[ch.add], ch.add, [&](uint32_t v) { if (v < C::V) vch[v] = (uint16_t)c; });
    }
    g.sync();
    if (g.rank == 0) {
#pragma unroll 1
        for (uint32_t c = 0; c < nc; c++) {
#pragma unroll 1
            for (int w = 0; w < 2; w++) {
                const uint32_t u = w ? chain[c].mufu : chain[c].add;
                const uint16_t key = own[u];
                f_value_operands(W, W.hdr[u], u, [&](uint32_t v) {
                    const uint32_t i = v < C::V ? W.defslot[v] : (uint32_t)F_NONE;
                    if (i != F_NONE && f_live(W, i) && key < rch[i]) rch[i] = key;
                });
            }
        }
    }
    g.sync();
    FFOR(g, s, n) if (s < n && f_live(W, s)) {
        const uint32_t key = own[s] < rch[s] ? own[s] : rch[s];
        if (key == F_NONE) continue;
        f_value_operands(W, W.hdr[s], s, [&](uint32_t v) { if (v < C::V && vch[v] != F_NONE) a_min32(&qmin[vch[v]], key); });
    }
    g.sync();
    FFOR(g, c, nc) if (c < nc) {
        const uint32_t q = qmin[c] < rch[chain[c].add] ? qmin[c] : rch[chain[c].add];
        if (q < crank[c]) f_fail(W, F_REDO + 35);
    }
    g.sync();
    if (!f_oks(g, W)) return;
    /* rewrite: ids by rank (_insert_reciprocal_bitcasts :863-888) */
    const uint32_t a0 = W.n_slots, v0 = W.next_vid, i0 = W.next_iid, l0 = W.n_log, e0 = W.n_ev;
    if (a0 + 2 * nc > C::I || v0 + 2 * nc > C::V || l0 + 2 * nc > C::L || e0 + nc > C::E) { if (g.rank == 0) f_fail(W, F_REDO + 41); g.sync(); return; }
    uint16_t *vmap = W.redirect;                     /* add result -> its float view */
    FFOR(g, v, nv) if (v < nv) vmap[v] = F_NONE;
    g.sync();
    FFOR(g, c, nc) if (c < nc) {
        const FChain ch = chain[c];
        const uint32_t r = crank[c], vi = v0 + 2 * r, vf = vi + 1, iid = i0 + 2 * r, sa = a0 + 2 * r;
        const cl_hdr ah = W.hdr[ch.add];
        W.alive[vi] = 1; W.norigin[vi] = (uint16_t)(2u << 14 | ch.rcp); W.usecnt[vi] = 1; W.defslot[vi] = (uint16_t)sa;
        W.alive[vf] = 1; W.norigin[vf] = (uint16_t)(3u << 14 | ch.addv); W.usecnt[vf] = 0; W.defslot[vf] = (uint16_t)(sa + 1);
        W.dlog[l0 + 2 * r].vid = vi; W.dlog[l0 + 2 * r].iid = (int32_t)iid;
        W.dlog[l0 + 2 * r + 1].vid = vf; W.dlog[l0 + 2 * r + 1].iid = (int32_t)(iid + 1);
        const unsigned u0 = use0(ah);
#pragma unroll 1
        for (unsigned k = 0; k < ah.n_uses; k++) {
            const opnd x = f_slot(W, ch.add, u0 + k);
            if (is_value(x) && x.pay == ch.rcp) W.pay[ch.add * 8 + u0 + k] = vi;
        }
        vmap[ch.addv] = (uint16_t)vf;
#pragma unroll 1
        for (unsigned q = 0; q < 2; q++) {
            const uint32_t s = sa + q;
            cl_hdr h;
            h.iid = iid + q; h.op = CL_OP_BITCAST; h.modset = q ? CL_MS_I2F : CL_MS_F2I;
            h.n_defs = 1; h.n_aux = 0; h.n_uses = 1; h.flags = 0; h.ext = 0;
            W.hdr[s] = h;
#pragma unroll 1
            for (unsigned k = 0; k < 8; k++) { W.tag[s * 8 + k] = k < 2 ? (uint16_t)CL_K_VALUE : (uint16_t)0; W.pay[s * 8 + k] = 0; }
            W.pay[s * 8] = vi + q; W.pay[s * 8 + 1] = q ? ch.addv : ch.rcp;
            W.sflag[s] = (uint8_t)(SF_LIVE | SF_PURE | SF_INS | f_cls(*e.P, 0, CL_OP_BITCAST) << SF_CLS_SHIFT);
            W.nxt[s] = q ? F_NONE : (uint16_t)(s + 1);
            W.sblk[s] = W.sblk[ch.add];
            W.posof[s] = W.posof[ch.add];
        }
        f_inc_use(W, ch.addv);                         /* the BITCAST.I2F reads the add's result */
        const uint32_t ap = W.posof[ch.add];
        W.insslot[ap] = (uint16_t)sa; W.inscnt[ap] = (uint8_t)(1u | INS_AFTER);
        cl_event ev; ev.func = W.f; ev.seq = 1u << 28; ev.kind = CL_EV_BOUNDARY; ev.idx = r; ev.a = ch.rcp; ev.b = ah.iid; ev.c = 0; ev.d = 0;
        W.ev[e0 + r] = ev;
    }
    g.sync();
    /* every user of an add result (top-level uses only :878-883) reads the float view */
    FFOR(g, s, a0) if (s < a0 && f_live(W, s)) {
        const cl_hdr h = W.hdr[s];
        const unsigned u0 = use0(h);
#pragma unroll 1
        for (unsigned k = 0; k < h.n_uses; k++) {
            const opnd x = f_slot(W, s, u0 + k);
            if (is_value(x) && x.pay < nv && vmap[x.pay] != F_NONE) {
                const uint32_t vf = vmap[x.pay];
                W.pay[s * 8 + u0 + k] = vf;
                f_inc_use(W, vf);
                a_sub(&W.usecnt[x.pay], 1u);           /* never reaches zero: the bitcast keeps one */
            }
        }
    }
    g.sync();
    if (g.rank == 0) {
        W.n_slots = a0 + 2 * nc; W.next_vid = v0 + 2 * nc; W.next_iid = i0 + 2 * nc; W.n_log = l0 + 2 * nc; W.n_ev = e0 + nc; W.dirty = 1;
        /* a float view nobody reads is dead on arrival (removed by the next remove_dead_pseudo) */
#pragma unroll 1
        for (uint32_t c = 0; c < nc; c++) if (W.usecnt[v0 + 2 * c + 1] == 0) f_push_wl(W, a0 + 2 * c + 1);
    }
    g.sync();
    f_rebuild(g, W);
}

/* CL_ORG_* code of a value created on the device (FW::norigin)                */
CLD uint32_t f_origin(uint16_t o) { const uint32_t k = o >> 14; return k == 1 ? (uint32_t)CL_ORG_PAIR : (k << 28 | (o & 0x3FFFu)); }

/* ------------------------------------------------------------------ store */
/* the result goes, once, to an atomically reserved place of every output
 * stream (completion order; the run densifies to function order afterwards)  */
template <class G, class C> CLF void f_store(const G &g, FW<C> &W, const FEnv &e, const cl_event *mev) {
    const KArgs &a = *e.a;
    const uint32_t n = W.n_pos, nv = W.next_vid, nq = W.nq_in + W.n_newimm, f = W.f;
    const uint32_t n_mev = mev ? W.n_mev : 0u, n_ev = W.n_ev + n_mev;
    if (g.rank == 0) {
        W.r_inst = (uint32_t)a_add64(&a.cursor[CUR_INST], n);
        W.r_imm = (uint32_t)a_add64(&a.cursor[CUR_IMM], nq);
        W.r_val = (uint32_t)a_add64(&a.cursor[CUR_VAL], nv);
        W.r_ev = (uint32_t)a_add64(&a.cursor[CUR_EV], n_ev);
    }
    g.sync();
    const uint32_t r_inst = W.r_inst, r_imm = W.r_imm, r_val = W.r_val, r_ev = W.r_ev;
    const bool fits = (unsigned long long)r_inst + n <= a.cap[CUR_INST] && (unsigned long long)r_imm + nq <= a.cap[CUR_IMM] &&
                      (unsigned long long)r_val + nv <= a.cap[CUR_VAL] && (unsigned long long)r_ev + n_ev <= a.cap[CUR_EV];
    if (g.rank == 0) {
        FuncOut o;
        o.f.next_vid = nv; o.f.next_iid = W.next_iid; o.f.next_temp_reg = W.next_temp;
        o.f.arch = (uint8_t)W.arch; o.f.status = (uint8_t)(fits ? CL_ST_OK : CL_ST_CAPACITY); o.f.reserved = 0;
        o.inst_start = r_inst; o.n_inst = fits ? n : 0; o.imm_start = r_imm; o.n_imm = fits ? nq : 0;
        o.val_start = r_val; o.ev_start = r_ev; o.n_ev = fits ? n_ev : 0; o.pad = 0;
        a.o_func[f] = o;
    }
    const uint32_t b0 = W.b0, nb = W.nb;
    FFOR(g, b, nb) if (b < nb) {
        a.o_blk[b0 + b] = W.blk[b];
        a.o_blk_start[b0 + b] = fits ? r_inst + W.bo[b] : 0u;
        a.o_blk_cnt[b0 + b] = fits ? (uint32_t)(W.bo[b + 1] - W.bo[b]) : 0u;
    }
    FFOR(g, m, W.n_mem) if (m < W.n_mem) a.o_mem[W.m0 + m] = W.mem[m];
    if (!fits) return;
    {
        const uint16_t *o = W.ord[W.cur];
        uint4 *dh = (uint4 *)(a.o_hdr + r_inst), *dt = (uint4 *)(a.o_tag + (size_t)r_inst * 8), *dp = (uint4 *)(a.o_pay + (size_t)r_inst * 8);
        const uint4 *sh = (const uint4 *)W.hdr, *st = (const uint4 *)W.tag, *sp = (const uint4 *)W.pay;
        FFOR(g, p, n) if (p < n) { const uint32_t s = o[p]; dh[p] = sh[s]; dt[p] = st[s]; }
        FFOR(g, q, 2 * n) if (q < 2 * n) { const uint32_t s = o[q >> 1]; dp[q] = sp[2 * s + (q & 1u)]; }
    }
    {
        const cl_imm *src = a.in.imm + W.q0;
        FFOR(g, q, nq) if (q < nq) a.o_imm[r_imm + q] = q < W.nq_in ? src[q] : W.newimm[q - W.nq_in];
    }
    {
        const int32_t *sd = a.in.val_def_iid + W.v0;
        FFOR(g, v, nv) if (v < nv) {
            a.o_alive[r_val + v] = W.alive[v];
            a.o_def_iid[r_val + v] = v < W.nv_in ? sd[v] : -1;
            a.o_origin[r_val + v] = v < W.nv_in ? (uint32_t)CL_ORG_HOST : f_origin(W.norigin[v]);
        }
    }
    FFOR(g, k, W.n_ev) if (k < W.n_ev) a.o_ev[r_ev + k] = W.ev[k];
    FFOR(g, k, n_mev) if (k < n_mev) a.o_ev[r_ev + W.n_ev + k] = mev[k];
    g.sync();
    /* def_iid updates in program order (a value redefined twice keeps the last) */
    if (g.rank == 0) for (uint32_t k = 0; k < W.n_log; k++) a.o_def_iid[r_val + W.dlog[k].vid] = W.dlog[k].iid;
}

/* ------------------------------------------------------------ the CTA's loop */
template <class C> CLHD size_t f_scratch_bytes(uint32_t mev_cap) { return (size_t)(C::E + mev_cap) * sizeof(cl_event) + (size_t)C::L * sizeof(FDLog); }
struct FLoop {
    /* work of this class: entries [bounds[0], bounds[1]) of the size-sorted function list (device side counting
     * sort, fused.cu), then what the class before could not take (list2, n_list2 on the device)              */
    const uint32_t *list; const uint32_t *bounds;
    const uint32_t *list2; const uint32_t *n_list2_ptr;
    uint32_t *counter;
    uint32_t *next_list, *next_count;       /* functions too large for this class (null: retry lists)           */
    uint8_t *scr; uint32_t mev_cap;         /* per group global scratch: C::E events of the function, mev_cap match events (emit_matches), C::L def_iid updates */
};

/* Persistent loop of the groups of one CTA over the functions of their size
 * class.  The groups take one function each and walk through the passes in
 * LOCK STEP (a CTA barrier between two phases): the stage is a few hundred KB
 * of code, far beyond the instruction cache, and warps that each sit in a
 * different phase of a different function spend their time on instruction
 * fetch misses (measured: 2 M cycles per function free-running).  In lock
 * step an SM runs one phase's code at a time for all its resident functions.
 * What does not fit the class goes to the next class's list, hand-backs to the
 * general kernel.                                                            */
/* one round of _apply_patterns for the resident functions of the CTA; `on`: this group takes part
 * (with its own table: the pooled items are per pattern, and the two tables share no pattern).
 * Returns the group's number of successful rewrites.                                             */
template <class G, class C> CLF uint32_t f_apply_step(const G &g, FW<C> &W, const FEnv &e, const FCtx<C> &x, bool on, unsigned table, uint32_t phase,
                                                      cl_event *mv, uint32_t mev_cap, bool match_only) {
    if (on) {
        if (f_rd(g, &W.dirty)) f_rebuild(g, W);
        f_prof(g, W, PF_MOVE);
        f_match_prep(g, W, e, x, table);
    } else
        f_match_idle(g, x);
    f_match_pooled(x, e);
    f_prof(g, W, PF_MATCH);
    const uint32_t nm = on && f_oks(g, W) ? f_rd(g, &W.n_mt) : 0u;
    if (nm) {
        f_select(g, W);
        if (mv && f_oks(g, W)) f_emit_matches(g, W, e, phase, mv, mev_cap);
    }
    f_prof(g, W, PF_SELECT);
    const bool plan = nm != 0 && !match_only && f_oks(g, W);
    f_plan_prep(g, W, x, plan);
    f_plan_pooled(x, e);
    uint32_t n = 0;
    if (plan) n = f_plan_commit(g, W, e, table, phase);
    f_prof(g, W, PF_PLAN);
    return n;
}

/* Persistent loop of the groups of one CTA over the functions of their size
 * class.  Every group holds one function and is in one of a few states; an
 * iteration of the loop is one apply step (match, select, plan, commit) taken by
 * all groups TOGETHER, whatever round their function is in, followed by what
 * each group's state asks for (pack folding, or the end of the function: dead
 * code, tags, store, and the next function's load, def-use and reciprocal pass).
 * Lock step, because the stage is far more code than the instruction cache
 * holds: free-running warps, each in another phase of another function, spent
 * their time on instruction fetch (measured: 2 M cycles per function; 0.3 M in
 * lock step).  A group never waits for another function's later rounds: it
 * finishes its own and joins the next step with a new one.                     */
enum { FST_EMPTY = 0, FST_XMAD, FST_ROUND, FST_MATCH_ONLY };
template <class G, class C> CLF void f_loop(const G &g, FW<C> &W, const FEnv &e, const FCtx<C> &x, const FLoop &L, uint32_t group) {
    const KArgs &a = *e.a;
    const uint32_t lo1 = L.bounds[0], n1 = L.bounds[1] - lo1, n2 = L.n_list2_ptr ? *L.n_list2_ptr : 0u, n_list = n1 + n2;
    unsigned long long n_in = 0, n_out = 0, n_ev = 0;
    if (g.rank == 0) {
#pragma unroll 1
        for (int k = 0; k < PF__N; k++) W.prof[k] = 0;
        W.prof_t = now();
        uint8_t *scr = L.scr + (size_t)group * f_scratch_bytes<C>(L.mev_cap);
        W.ev = (cl_event *)scr;
        W.dlog = (FDLog *)(scr + (size_t)(C::E + L.mev_cap) * sizeof(cl_event));
    }
    g.sync();
    cl_event *mev = L.mev_cap ? W.ev + C::E : nullptr;
    const bool match_only = (a.passes & CL_PASS_MATCH_ONLY) != 0;
    const bool emit = a.emit_matches || match_only;
    cl_event *mv = emit ? mev : nullptr;
    int st = FST_EMPTY;
    uint32_t round = 0, f = 0;
    bool exhausted = false;
    /* the function is finished (ok) or given up (hand-back / next class): the group is free again */
    auto leave = [&](bool ok) {
        if (ok) {
            if (f_rd(g, &W.dirty)) f_rebuild(g, W);
            f_prof(g, W, PF_MOVE);
            f_store(g, W, e, mv);
            f_prof(g, W, PF_STORE);
            g.sync();
            FFOR(g, k, 64) if (k < 64 && W.fstat[k]) a_add64(&a.stats[k], W.fstat[k]);
            if (g.rank == 0) { n_in += W.n_in; n_out += W.n_pos; n_ev += W.n_ev + (mv ? W.n_mev : 0u); }
#if !CL_DEV
            if (getenv("CL_FUSED_STATS")) fprintf(stderr, "fused done: n_in %u slots %u out %u nv_in %u nv %u newimm %u log %u ev %u\n", W.n_in, W.n_slots, W.n_pos, W.nv_in, W.next_vid, W.n_newimm, W.n_log, W.n_ev);
#endif
        } else {
#if !CL_DEV
            if (getenv("CL_FUSED_DEBUG")) fprintf(stderr, "fused hand-back: function %u (%u records) reason %u\n", f, W.n_in, W.fail);
#endif
            if (g.rank == 0) {
                /* outgrew its slice while running: the next class has more room; else the general kernel */
                if (W.fail > F_REDO + 40 && W.fail < F_REDO + 60 && L.next_list) L.next_list[a_add(L.next_count, 1u)] = f;
                else {
                    const cl_corpus &in = a.in;
                    const uint32_t n = in.blk_off[in.func_blk_off[f + 1]] - in.blk_off[in.func_blk_off[f]];
                    if (n > a.small_max) a.retry_big_list[a_add(a.retry_big_count, 1u)] = f;
                    else a.retry_list[a_add(a.retry_count, 1u)] = f;
                }
            }
        }
        g.sync();
        st = FST_EMPTY;
    };
    /* end of the function's passes: remove_dead_pseudo of apply_aggregations, tag_cuda_objects */
    auto finish = [&]() {
        if ((a.passes & CL_PASS_AGGREGATE) && f_oks(g, W)) f_dce(g, W);
        f_prof(g, W, PF_DCE);
        if ((a.passes & CL_PASS_TAG) && f_oks(g, W)) f_tag(g, W, e);
        f_prof(g, W, PF_TAG);
        leave(f_oks(g, W));
    };
    /* normalize_reciprocal, then the first aggregation round (or the end) */
    auto after_xmad = [&]() {
        if ((a.passes & CL_PASS_RECIPROCAL) && (f_rd(g, &W.flags) & FF_RCP) && f_oks(g, W)) {
            if (f_rd(g, &W.dirty)) f_rebuild(g, W);
            f_reciprocal(g, W, e);
        }
        f_prof(g, W, PF_RECIP);
        if (!f_oks(g, W)) { leave(false); return; }
        if ((a.passes & CL_PASS_AGGREGATE) && a.max_rounds) { st = FST_ROUND; round = 0; }
        else finish();
    };
#pragma unroll 1
    for (;;) {
        /* ---- a free group takes the next function of its class */
        if (st == FST_EMPTY && !exhausted) {
            g.sync();
            if (g.rank == 0) W.work = a_add(L.counter, 1u);
            g.sync();
            const uint32_t w = f_rd(g, &W.work);
            f_prof(g, W, PF_SETUP);
            if (w >= n_list) exhausted = true;
            else {
                f = w < n1 ? L.list[lo1 + w] : L.list2[w - n1];
                if (!f_load(g, W, e, f)) {
                    if (g.rank == 0) {           /* too large for this class */
                        if (L.next_list) L.next_list[a_add(L.next_count, 1u)] = f;
                        else {
                            const cl_corpus &in = a.in;
                            const uint32_t n = in.blk_off[in.func_blk_off[f + 1]] - in.blk_off[in.func_blk_off[f]];
                            if (n > a.small_max) a.retry_big_list[a_add(a.retry_big_count, 1u)] = f;
                            else a.retry_list[a_add(a.retry_count, 1u)] = f;
                        }
                    }
                } else {
                    f_prof(g, W, PF_LOAD);
                    const bool xm = (a.passes & CL_PASS_XMAD) && W.arch == CL_ARCH_SM52;
                    const unsigned table = match_only ? ((a.passes & CL_PASS_MATCH_XMAD) ? 1u : 0u) : (xm ? 1u : 0u);
                    if (g.rank == 0 && emit && !mev) f_fail(W, F_REDO + 23);
                    g.sync();
                    if (f_oks(g, W)) f_index(g, W, e, table);
                    f_prof(g, W, PF_USECOUNT);
                    if (!f_oks(g, W)) leave(false);
                    else if (match_only) { st = FST_MATCH_ONLY; round = table; }
                    else if (xm) st = FST_XMAD;
                    else after_xmad();
                }
            }
        }
        if (!f_cta_or(st != FST_EMPTY || !exhausted)) break;
        /* ---- one apply step, all groups together */
        const bool on = st != FST_EMPTY;
        const unsigned table = st == FST_XMAD ? 1u : st == FST_MATCH_ONLY ? round : 0u;
        const uint32_t phase = st == FST_ROUND ? 2 + round : 0u;
        uint32_t n = f_apply_step(g, W, e, x, on, table, phase, mv, L.mev_cap, st == FST_MATCH_ONLY);
        /* ---- what the group's state asks for */
        if (!on) continue;
        if (!f_oks(g, W)) { leave(false); continue; }
        if (st == FST_MATCH_ONLY) { leave(true); continue; }
        if (st == FST_XMAD) {                     /* normalize_xmad (patterns.py:805-810): one round, then dead code */
            f_dce(g, W);
            if ((a.passes & (CL_PASS_AGGREGATE | CL_PASS_RECIPROCAL)) && f_oks(g, W)) f_reclass(g, W, e, 0);
            f_prof(g, W, PF_DCE);
            if (!f_oks(g, W)) { leave(false); continue; }
            after_xmad();
            continue;
        }
        /* apply_aggregations (patterns.py:794-802): up to max_rounds of (_apply_patterns + simplify_packs) */
        n += f_simplify(g, W, e);
        f_prof(g, W, PF_SIMPLIFY);
        if (!f_oks(g, W)) { leave(false); continue; }
        round++;
        if (!n || round >= a.max_rounds) finish();
    }
    if (g.rank == 0) {
        a_add64(&a.stats[64], n_in); a_add64(&a.stats[65], n_out); a_add64(&a.stats[66], n_ev);
        unsigned long long tot = 0;
#pragma unroll 1
        for (int k = 1; k < PF__N; k++) { tot += W.prof[k]; if (W.prof[k]) a_add64(&a.prof[k], W.prof[k]); }
        a_add64(&a.prof[PF_TOTAL], tot);
    }
}

} /* namespace clk */

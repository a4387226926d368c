/* core.cuh -- the device algorithm of the normalisation + pattern-aggregation
 * path: one cooperative thread *group* (a warp for small functions, a whole
 * CTA for large ones) keeps one function resident in a gap buffer (shared
 * memory when it fits, L2-resident scratch otherwise) and takes it through
 *
 *   seed scan -> tuple unification -> overlap selection -> rewrite planning
 *   (count / exclusive scan / emit) -> pack simplification -> dead-pseudo
 *   elimination -> reciprocal normalisation -> CUDA-object tagging
 *
 * so that HBM sees one read of the input stream and one write of the result.
 * Semantics are those of the reference (cited per function, paths relative to
 * /root/reference/pkg/src/sasslift/); results are bit-exact with oracle/.
 *
 * The code is written against a small `Grp` interface (rank/size/sync/scan)
 * and plain generic pointers, so the same source also compiles as ordinary
 * C++ with a one-lane group (CL_SIM) -- used only by tests/sim to debug the
 * logic on machines without a GPU; the package never loads that build.
 */
#pragma once
#include "../../include/culifter.h"
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <stdlib.h>

#if defined(__CUDACC__) && !defined(CL_SIM)
#define CL_DEV 1
#define CLD __device__ __forceinline__
#define CLF __device__ __noinline__
#define CLN __device__ __noinline__
#define CLHD __host__ __device__ inline
#define CLM static __device__ __forceinline__
#define CLMEM __device__ __forceinline__
#else
#define CL_DEV 0
#define CLD static inline
#define CLF static
#define CLN static
#define CLHD static inline
#define CLM static inline
#define CLMEM inline
struct alignas(16) uint4 { uint32_t x, y, z, w; };
#endif

namespace clk {

static constexpr uint32_t NONE32 = 0xFFFFFFFFu;
static constexpr unsigned long long NONE64 = ~0ull;

/* ----------------------------------------------------------------- atomics */
CLD uint32_t a_add(uint32_t *p, uint32_t v) {
#if CL_DEV
    return atomicAdd(p, v);
#else
    uint32_t o = *p; *p += v; return o;
#endif
}
CLD void a_cas0(uint32_t *p, uint32_t v) {      /* set if still zero */
#if CL_DEV
    atomicCAS(p, 0u, v);
#else
    if (*p == 0) *p = v;
#endif
}
CLD uint32_t a_sub(uint32_t *p, uint32_t v) {
#if CL_DEV
    return atomicSub(p, v);
#else
    uint32_t o = *p; *p -= v; return o;
#endif
}
CLD void a_min64(unsigned long long *p, unsigned long long v) {
#if CL_DEV
    atomicMin(p, v);
#else
    if (v < *p) *p = v;
#endif
}
CLD void a_min32(uint32_t *p, uint32_t v) {
#if CL_DEV
    atomicMin(p, v);
#else
    if (v < *p) *p = v;
#endif
}
CLD uint32_t a_or(uint32_t *p, uint32_t v) {
#if CL_DEV
    return atomicOr(p, v);
#else
    uint32_t o = *p; *p |= v; return o;
#endif
}
/* append to a list whose cursor is *counter: one atomic per warp for the lanes that call it together */
CLD uint32_t a_append(uint32_t *counter) {
#if CL_DEV
    const unsigned act = __activemask();
    const unsigned lane = threadIdx.x & 31u;
    const int lead = __ffs((int)act) - 1;
    uint32_t base = 0;
    if ((int)lane == lead) base = atomicAdd(counter, (uint32_t)__popc(act));
    base = __shfl_sync(act, base, lead);
    return base + (uint32_t)__popc(act & ((1u << lane) - 1u));
#else
    return (*counter)++;
#endif
}
CLD unsigned long long a_add64(unsigned long long *p, unsigned long long v) {
#if CL_DEV
    return atomicAdd(p, v);
#else
    unsigned long long o = *p; *p += v; return o;
#endif
}

/* ---------------------------------------------------------------- profiling */
/* cycle counters per phase, accumulated by lane 0 of every group (cheap, always on);
 * cl_debug_profile() returns their sum over all groups                         */
enum { PF_TOTAL = 0, PF_LOAD, PF_STORE, PF_USECOUNT, PF_SEED, PF_MATCH, PF_SELECT, PF_PLAN, PF_EMIT, PF_MOVE,
       PF_SIMPLIFY, PF_DCE, PF_RECIP, PF_TAG, PF_SETUP, PF__N = 16 };
CLD unsigned long long now() {
#if CL_DEV
    return clock64();
#else
    return 0;
#endif
}
struct Prof {
    unsigned long long *acc, t0; bool on;
    CLMEM Prof(unsigned long long *a, int slot, bool lane0) : acc(a + slot), t0(0), on(lane0) { if (on) t0 = now(); }
    CLMEM ~Prof() { if (on) *acc += now() - t0; }
};
#ifdef CL_PROFILE
#define PROF(g, s, slot) Prof _prof_##slot((s).prof, slot, (g).rank == 0)
#else
#define PROF(g, s, slot) do { } while (0)      /* build with -DCL_PROFILE for the per-phase cycle counters */
#endif

/* ------------------------------------------------------------------ groups */
/* NW = warps per group.  NW == 1: the group is a warp (several independent
 * groups per CTA).  NW > 1: the group is the whole CTA.  NW == 0: host.     */
template <int NW> struct Grp {
    static constexpr uint32_t THREADS = NW * 32;
    uint32_t rank, size;
    uint32_t *red;             /* NW > 1: shared scratch, NW + 2 words         */
#if CL_DEV
    CLD void sync() const { if (NW == 1) __syncwarp(); else __syncthreads(); }
    /* second level of the CTA scans: warp 0 turns the per-warp totals in red[0 .. NW) into exclusive
     * prefixes (in place) and the grand total in red[NW]; callers sync before and after            */
    CLD void scan_warp_totals() const {
        if ((rank >> 5) == 0) {
            const uint32_t lane = rank & 31u;
            const uint32_t t = lane < (uint32_t)NW ? red[lane] : 0u;
            uint32_t v = t;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, v, d);
                if (lane >= (uint32_t)d) v += u;
            }
            if (lane < (uint32_t)NW) red[lane] = v - t;
            if (lane == 31) red[NW] = v;
        }
    }
    CLD uint32_t exscan(uint32_t x, uint32_t &total) const {
        const uint32_t lane = rank & 31u;
        uint32_t v = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, d);
            if (lane >= (uint32_t)d) v += t;
        }
        if (NW == 1) { total = __shfl_sync(0xFFFFFFFFu, v, 31); return v - x; }
        const uint32_t w = rank >> 5;
        if (lane == 31) red[w] = v;
        __syncthreads();
        scan_warp_totals();
        __syncthreads();
        /* red[w] is rewritten only by warp w itself (next call) and red[NW] only after the next call's
         * first barrier: no trailing barrier needed                                               */
        total = red[NW];
        return red[w] + v - x;
    }
    /* ballot + popc compaction offsets */
    CLD uint32_t flag_exscan(bool f, uint32_t &total) const {
        const uint32_t lane = rank & 31u;
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, f);
        const uint32_t mine = __popc(b & ((1u << lane) - 1u));
        if (NW == 1) { total = __popc(b); return mine; }
        const uint32_t w = rank >> 5;
        if (lane == 0) red[w] = __popc(b);
        __syncthreads();
        scan_warp_totals();
        __syncthreads();
        total = red[NW];
        return red[w] + mine;
    }
    CLD bool any(bool f) const {
        if (NW == 1) return __any_sync(0xFFFFFFFFu, f);
        return __syncthreads_or(f) != 0;
    }
    CLD uint32_t sum(uint32_t x) const { uint32_t t; exscan(x, t); return t; }
    CLD uint32_t bcast0(uint32_t x) const {
        if (NW == 1) return __shfl_sync(0xFFFFFFFFu, x, 0);
        if (rank == 0) red[NW + 1] = x;
        __syncthreads();
        uint32_t r = red[NW + 1];
        __syncthreads();
        return r;
    }
#endif
};

/* NW == 0: a group of one lane.  On the host it is the CL_SIM debug build; on
 * the device it is the thread-per-function kernel (32 independent functions
 * per warp: every lane is busy, the collectives are identities).            */
template <> struct Grp<0> {
    static constexpr uint32_t THREADS = 1;
    uint32_t rank, size;
    uint32_t *red;
    CLMEM void sync() const {}
    CLMEM uint32_t exscan(uint32_t x, uint32_t &total) const { total = x; return 0; }
    CLMEM uint32_t flag_exscan(bool f, uint32_t &total) const { total = f; return 0; }
    CLMEM bool any(bool f) const { return f; }
    CLMEM uint32_t sum(uint32_t x) const { return x; }
    CLMEM uint32_t bcast0(uint32_t x) const { return x; }
};

/* uniform strided loop: every lane runs every iteration (collectives inside
 * are legal); `i < n` guards the work.                                       */
#define GFOR(g, i, n) for (uint32_t _b##i = 0, i = (g).rank; _b##i < (n); _b##i += (g).size, i += (g).size)

/* ------------------------------------------------------------ data model */
struct opnd { uint16_t tag; uint32_t pay; };
struct alignas(16) Rec { cl_hdr h; uint16_t tag[8]; uint32_t pay[8]; };
struct Planes { cl_hdr *hdr; uint16_t *tag; uint32_t *pay; };

struct okey { uint32_t cls; unsigned long long v; };
enum { KC_NONE = 0, KC_V, KC_IMM, KC_RZ, KC_PT, KC_P, KC_CM, KC_R, KC_UR, KC_SR, KC_OTHER, KC_MOD };
static constexpr int NBIND = CL_MAX_VARS + CL_MAX_GROUPS;
struct Bind { okey var[NBIND]; };

struct MatchRec {              /* Match (patterns.py:100-106) on block positions */
    uint8_t pat, n, state, pad;
    uint32_t pos[3];
    uint32_t seq;              /* pattern << 20 | tuple rank: list order          */
};
enum { MS_UNDECIDED = 0, MS_SELECTED = 1, MS_REJECTED = 2 };

struct SelRec {                /* selected match, function wide                  */
    uint8_t pat, n, pad0, pad1;
    uint32_t blk;              /* block index                                    */
    uint32_t pos[3];           /* block-relative positions                       */
};
struct XRec {                  /* bitcast inserted by the reciprocal pass        */
    Rec r;
    uint32_t anchor;           /* stream position of the add                     */
    uint32_t order;            /* index in its anchor's before / after list      */
    uint32_t after;
    uint32_t next;             /* next extra user of the same value              */
};

/* opcode classes of the seed scan: distinct head opcodes of one table        */
static constexpr int MAX_CLS = 12;

struct Caps {                  /* capacities of one group's work memory          */
    uint32_t I;                /* records in the gap buffer                      */
    uint32_t V;                /* values                                         */
    uint32_t B;                /* blocks                                         */
    uint32_t M;                /* raw matches of one block                       */
    uint32_t S;                /* selected matches of one function               */
    uint32_t Q;                /* immediates                                     */
    uint32_t E;                /* events                                         */
    uint32_t U;                /* use sites (reciprocal CSR)                     */
    uint32_t X;                /* inserted bitcasts                              */
};

struct FS {                    /* one function resident in a group's work memory */
    const cl_pattern_blob *pb;
    const cl_modset *ms;
    const uint8_t *opflags;    /* CL_OPF_* by opcode id (< CL_OP__COUNT)         */
    Caps cap;
    uint32_t f;                /* function index                                 */
    bool solo;                 /* one-lane group: private updates need no atomics */
    uint32_t arch;
    uint32_t *st;              /* group-shared status word (enum cl_status)      */
    uint32_t passes, max_rounds, emit_matches;
    /* stream: records [0, n) of S, blocks bo[0..nb]                           */
    Planes S;
    uint32_t n, nb;
    uint32_t *bo, *bo2;        /* [B + 1] block offsets / next round's           */
    cl_blk *blk;               /* [B] mutable copy (terminator operands)         */
    /* values */
    uint32_t *usecnt, *defpos; /* [V]                                            */
    uint8_t *alive;            /* [V]                                            */
    int32_t *def_iid;          /* [V]                                            */
    uint32_t *origin;          /* [V]                                            */
    uint32_t *redirect;        /* [V]  (also CSR offsets of the reciprocal pass) */
    uint32_t next_vid, next_iid, next_temp;
    uint32_t odd_defs;         /* some def slot is neither a value nor RZ/PT: no join */
    /* side tables */
    cl_imm *imm; uint32_t n_imm;
    cl_memref *mem; uint32_t n_mem;
    uint16_t *ext_tag; uint32_t *ext_pay; uint32_t n_ext;
    cl_event *ev; uint32_t *n_ev;       /* n_ev: one word of group-shared memory  */
    /* per position scratch [I] */
    uint8_t *keep, *inscnt, *clsid;
    uint32_t *outpos, *cand, *sel_at;
    uint32_t *cidx;            /* index of a position inside its seed class (aliases outpos) */
    unsigned long long *owner;
    /* per match scratch */
    MatchRec *mt;              /* [M]                                            */
    SelRec *sel;               /* [S]                                            */
    struct Stage *stage;       /* [S] staged rewrite of each selected match       */
    uint32_t *blk_sel;         /* [B + 1] selected-match range of each block     */
    /* reciprocal */
    uint32_t *site;            /* [U]                                            */
    XRec *xr;                  /* [X]                                            */
    uint32_t *xhead;           /* [V]                                            */
    uint32_t *root;            /* [V]                                            */
    /* statistics (group-private, flushed by the kernel)                       */
    uint32_t *st_matches, *st_selected, *st_rewrites, *st_refused;   /* [16] each */
    unsigned long long *prof;  /* [PF__N] group-private cycle counters              */
    /* seed classes of the current table */
    uint32_t n_cls;
    uint16_t cls_op[MAX_CLS];
    uint32_t cls_off[MAX_CLS + 1];
};

/* ---------------------------------------------------------- operand access */
CLD unsigned kind_of(uint16_t t) { return CL_T_KIND(t); }
CLD bool has_guard(const cl_hdr &h) { return (h.flags & CL_IF_GUARD) != 0; }
CLD unsigned def0(const cl_hdr &h) { return has_guard(h); }
CLD unsigned aux0(const cl_hdr &h) { return has_guard(h) + h.n_defs; }
CLD unsigned use0(const cl_hdr &h) { return has_guard(h) + h.n_defs + h.n_aux; }
CLN opnd get_slot(const FS &s, const cl_hdr &h, uint32_t i, unsigned k) {
    opnd o;
    if (h.flags & CL_IF_EXT) { o.tag = s.ext_tag[h.ext + k]; o.pay = s.ext_pay[h.ext + k]; }
    else { o.tag = s.S.tag[(size_t)i * 8 + k]; o.pay = s.S.pay[(size_t)i * 8 + k]; }
    return o;
}
CLN void set_slot(FS &s, const cl_hdr &h, uint32_t i, unsigned k, opnd o) {
    if (h.flags & CL_IF_EXT) { s.ext_tag[h.ext + k] = o.tag; s.ext_pay[h.ext + k] = o.pay; }
    else { s.S.tag[(size_t)i * 8 + k] = o.tag; s.S.pay[(size_t)i * 8 + k] = o.pay; }
}
CLD opnd get_use(const FS &s, const cl_hdr &h, uint32_t i, unsigned k) { return get_slot(s, h, i, use0(h) + k); }
CLD opnd get_def(const FS &s, const cl_hdr &h, uint32_t i, unsigned k) { return get_slot(s, h, i, def0(h) + k); }
CLD opnd get_aux(const FS &s, const cl_hdr &h, uint32_t i, unsigned k) { return get_slot(s, h, i, aux0(h) + k); }
CLD bool is_value(opnd o) { return kind_of(o.tag) == CL_K_VALUE; }
CLD bool is_zero(opnd o) { return kind_of(o.tag) == CL_K_RZ || kind_of(o.tag) == CL_K_URZ; }
CLD bool is_imm(opnd o) { return kind_of(o.tag) == CL_K_IMM; }
CLD bool is_none(opnd o) { return kind_of(o.tag) == CL_K_NONE; }
/* getattr(op, "negated"/"bitnot"/"half", default) of patterns.py:142-144     */
CLD bool o_neg(opnd o) { return (o.tag & CL_T_NEG) != 0; }
CLD bool o_not(opnd o) { return !is_imm(o) && (o.tag & CL_T_NOT) != 0; }
CLD unsigned o_half(opnd o) { return is_imm(o) ? 0u : CL_T_HALF(o.tag); }
CLD uint64_t modmask(const FS &s, const cl_hdr &h) { return s.ms[h.modset].mask; }
CLD bool has_mod(const FS &s, const cl_hdr &h, unsigned bit) { return (modmask(s, h) >> bit) & 1u; }
CLD opnd value_ref(uint32_t vid) { opnd o; o.tag = CL_K_VALUE; o.pay = vid; return o; }
CLD opnd strip(opnd o) { if (is_value(o)) o.tag &= (uint16_t)~(CL_T_NEG | CL_T_NOT); return o; }

/* value_operands (ssa.py:599-610): guard, uses, MemRef base/ureg             */
template <class F> CLD void for_value_operands(const FS &s, const cl_hdr &h, uint32_t i, F fn) {
    if (has_guard(h)) { opnd g = get_slot(s, h, i, 0); if (is_value(g)) fn(g.pay); }
    const unsigned u0 = use0(h);
    for (unsigned k = 0; k < h.n_uses; k++) {
        opnd u = get_slot(s, h, i, u0 + k);
        if (is_value(u)) fn(u.pay);
        else if (kind_of(u.tag) == CL_K_MEMREF) {
            const cl_memref &m = s.mem[u.pay];
            if (kind_of(m.base_tag) == CL_K_VALUE) fn(m.base_pay);
            if (kind_of(m.ureg_tag) == CL_K_VALUE) fn(m.ureg_pay);
        }
    }
}
template <class F> CLD void for_value_defs(const FS &s, const cl_hdr &h, uint32_t i, F fn) {
    const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
    for (unsigned k = 0; k < nd; k++) { opnd d = get_slot(s, h, i, d0 + k); if (is_value(d)) fn(d.pay); }
}

CLN void ld_rec(const FS &s, uint32_t i, Rec &r) {
    r.h = s.S.hdr[i];
    const uint4 *t = (const uint4 *)(s.S.tag + (size_t)i * 8);
    const uint4 *p = (const uint4 *)(s.S.pay + (size_t)i * 8);
    *(uint4 *)r.tag = t[0];
    ((uint4 *)r.pay)[0] = p[0];
    ((uint4 *)r.pay)[1] = p[1];
}
CLN void st_rec(FS &s, uint32_t i, const Rec &r) {
    s.S.hdr[i] = r.h;
    *(uint4 *)(s.S.tag + (size_t)i * 8) = *(const uint4 *)r.tag;
    ((uint4 *)(s.S.pay + (size_t)i * 8))[0] = ((const uint4 *)r.pay)[0];
    ((uint4 *)(s.S.pay + (size_t)i * 8))[1] = ((const uint4 *)r.pay)[1];
}

/* move n records from src to dst inside the gap buffer (any overlap)          */
template <class G> CLF void move_recs(const G &g, FS &s, uint32_t dst, uint32_t src, uint32_t n) {
    PROF(g, s, PF_MOVE);
    if (dst == src || n == 0) return;
    const uint32_t chunks = (n + g.size - 1) / g.size;
    for (uint32_t c = 0; c < chunks; c++) {
        const uint32_t cc = dst < src ? c : chunks - 1 - c;
        const uint32_t i = cc * g.size + g.rank;
        Rec r;
        if (i < n) ld_rec(s, src + i, r);
        g.sync();
        if (i < n) st_rec(s, dst + i, r);
        g.sync();
    }
}

/* updates of group-private data: atomic among the lanes of a group, plain for
 * a one-lane group (s.solo)                                                  */
CLD uint32_t p_add(const FS &s, uint32_t *p, uint32_t v) { if (s.solo) { const uint32_t o = *p; *p = o + v; return o; } return a_add(p, v); }
CLD uint32_t p_sub(const FS &s, uint32_t *p, uint32_t v) { if (s.solo) { const uint32_t o = *p; *p = o - v; return o; } return a_sub(p, v); }
CLD void p_min64(const FS &s, unsigned long long *p, unsigned long long v) { if (s.solo) { if (v < *p) *p = v; } else a_min64(p, v); }
CLD void p_min32(const FS &s, uint32_t *p, uint32_t v) { if (s.solo) { if (v < *p) *p = v; } else a_min32(p, v); }
/* first error wins; read it back only after a group sync                     */
CLD void fail(FS &s, uint32_t code) { if (s.solo) { if (!*s.st) *s.st = code; } else a_cas0(s.st, code); }
CLD uint32_t status(const FS &s) { return *(volatile uint32_t *)s.st; }

CLN void push_event(FS &s, uint32_t seq, uint32_t kind, uint32_t idx, uint32_t a, uint32_t b,
                    uint32_t c, uint32_t d) {
    uint32_t k = p_add(s, s.n_ev, 1u);
    if (k < s.cap.E) {
        cl_event e; e.func = s.f; e.seq = seq; e.kind = kind; e.idx = idx; e.a = a; e.b = b; e.c = c; e.d = d;
        s.ev[k] = e;
    } else
        fail(s, CL_ST_CAPACITY);            /* never a silently shortened event list: the function reports CapacityError */
}

/* ------------------------------------------------------------------ def-use */
/* Use counts (= len(du.users(vid)), terminator sites included) and the stream
 * position of each value's defining instruction (du.def_inst), ssa.py:613-636 */
template <class G> CLF void build_usecount(const G &g, FS &s) {
    PROF(g, s, PF_USECOUNT);
    GFOR(g, v, s.next_vid) if (v < s.next_vid) { s.usecnt[v] = 0; s.defpos[v] = NONE32; }
    g.sync();
    bool odd = false;
    GFOR(g, i, s.n) if (i < s.n) {
        const cl_hdr h = s.S.hdr[i];
        const unsigned d0 = def0(h), nd = (unsigned)h.n_defs + h.n_aux;
        for (unsigned k = 0; k < nd; k++) {
            const opnd d = get_slot(s, h, i, d0 + k);
            const unsigned kd = kind_of(d.tag);
            if (kd == CL_K_VALUE) { if (d.pay < s.cap.V) s.defpos[d.pay] = i; }
            else odd |= !(kd == CL_K_RZ || kd == CL_K_URZ || kd == CL_K_PRED);
        }
        for_value_operands(s, h, i, [&](uint32_t v) { if (v < s.cap.V) p_add(s, &s.usecnt[v], 1u); });
    }
    s.odd_defs = g.any(odd);
    GFOR(g, b, s.nb) if (b < s.nb)
        for (int k = 0; k < 2; k++)
            if (kind_of(s.blk[b].term_tag[k]) == CL_K_VALUE && s.blk[b].term_pay[k] < s.cap.V)
                p_add(s, &s.usecnt[s.blk[b].term_pay[k]], 1u);
    g.sync();
}

/* ----------------------------------------------------------------- matching */
/* operand_key (patterns.py:109-127)                                           */
CLN okey operand_key(const FS &s, opnd o) {
    okey k; k.cls = KC_OTHER; k.v = o.pay;
    switch (kind_of(o.tag)) {
    case CL_K_VALUE: k.cls = KC_V; break;
    case CL_K_IMM: k.cls = KC_IMM; k.v = s.imm[o.pay].bits; break;
    case CL_K_RZ: case CL_K_URZ: k.cls = KC_RZ; k.v = 0; break;
    case CL_K_PRED: if (o.pay == CL_PT_INDEX) { k.cls = KC_PT; k.v = 0; } else k.cls = KC_P; break;
    case CL_K_CONSTMEM: k.cls = KC_CM; break;
    case CL_K_REG: k.cls = KC_R; break;
    case CL_K_UREG: k.cls = KC_UR; break;
    case CL_K_SREG: k.cls = KC_SR; break;
    default: break;
    }
    return k;
}
CLN bool memref_equal(const FS &s, uint32_t a, uint32_t b) {
    const cl_memref &x = s.mem[a], &y = s.mem[b];
    if (x.base_tag != y.base_tag || x.ureg_tag != y.ureg_tag) return false;
    if (kind_of(x.base_tag) != CL_K_NONE && x.base_pay != y.base_pay) return false;
    if (kind_of(x.ureg_tag) != CL_K_NONE && x.ureg_pay != y.ureg_pay) return false;
    return x.off_hi == y.off_hi && x.off_lo == y.off_lo;
}
CLD bool key_equal(const FS &s, okey a, okey b) {
    if (a.cls != b.cls) return false;
    if (a.cls == KC_OTHER) return memref_equal(s, (uint32_t)a.v, (uint32_t)b.v);
    return a.v == b.v;
}
/* Bindings.bind (patterns.py:93-97)                                           */
CLD bool bind(const FS &s, Bind &b, unsigned name, okey k) {
    if (b.var[name].cls != KC_NONE && !key_equal(s, b.var[name], k)) return false;
    b.var[name] = k;
    return true;
}
/* _match_slot (patterns.py:130-152)                                           */
CLN bool match_slot(const FS &s, const cl_slot &sl, opnd o, Bind &b) {
    switch (sl.kind) {
    case CL_S_ANY: return true;
    case CL_S_RZ: return is_zero(o);
    case CL_S_PT:
        if (!(kind_of(o.tag) == CL_K_PRED && o.pay == CL_PT_INDEX)) return false;
        return sl.neg == 0 || o_neg(o) == (sl.neg == 2);
    case CL_S_IMM: return is_imm(o) && s.imm[o.pay].bits == sl.imm;
    case CL_S_VAR:
        if (sl.neg && o_neg(o) != (sl.neg == 2)) return false;
        if (sl.bitnot && o_not(o) != (sl.bitnot == 2)) return false;
        if (sl.half && o_half(o) != sl.half) return false;
        return bind(s, b, sl.var, operand_key(s, o));
    }
    return false;
}
/* _match_opcode + _unify (patterns.py:155-178)                                */
CLN bool match_inst(const FS &s, const cl_template &t, const cl_hdr &h, uint32_t i, Bind &b) {
    if (h.op != t.op) return false;
    const cl_modset &ms = s.ms[h.modset];
    if ((ms.mask & t.mods_all) != t.mods_all) return false;
    if (ms.mask & t.mods_none) return false;
    for (unsigned k = 0; k < t.n_modvars; k++) {
        const uint8_t got = ms.first[t.modvar_group[k]];
        okey key; key.cls = KC_MOD; key.v = got;
        if (got == 0xFF || !bind(s, b, CL_MAX_VARS + t.modvar_var[k], key)) return false;
    }
    if (t.n_defs != h.n_defs || t.n_aux != h.n_aux || t.n_uses != h.n_uses) return false;
    const unsigned n = (unsigned)t.n_defs + t.n_aux + t.n_uses, g0 = has_guard(h);
    if (h.flags & CL_IF_EXT) return false;          /* > 8 slots never equals a template's arity */
    for (unsigned k = 0; k < n; k++)
        if (!match_slot(s, t.slot[k], get_slot(s, h, i, g0 + k), b)) return false;
    return true;
}
/* _connected (patterns.py:219-238)                                            */
CLF bool connected(const FS &s, const uint32_t *idx, unsigned n) {
    if (n == 1) return true;
    uint32_t vals[CL_MAX_TEMPLATES][24];
    unsigned cnt[CL_MAX_TEMPLATES];
    for (unsigned t = 0; t < n; t++) {
        unsigned c = 0;
        const cl_hdr h = s.S.hdr[idx[t]];
        for_value_defs(s, h, idx[t], [&](uint32_t v) { if (c < 24) vals[t][c++] = v; });
        for_value_operands(s, h, idx[t], [&](uint32_t v) { if (c < 24) vals[t][c++] = v; });
        cnt[t] = c;
    }
    unsigned linked = 1;
    for (bool changed = true; changed;) {
        changed = false;
        for (unsigned i = 0; i < n; i++) {
            if (linked >> i & 1) continue;
            bool hit = false;
            for (unsigned j = 0; j < n && !hit; j++) {
                if (!(linked >> j & 1)) continue;
                for (unsigned a = 0; a < cnt[i] && !hit; a++)
                    for (unsigned c = 0; c < cnt[j]; c++) if (vals[i][a] == vals[j][c]) { hit = true; break; }
            }
            if (hit) { linked |= 1u << i; changed = true; }
        }
    }
    return linked == (1u << n) - 1u;
}
/* one candidate tuple of match_patterns (patterns.py:199-215); idx = stream
 * positions, strictly increasing order already checked by the caller         */
CLF bool check_tuple(const FS &s, const cl_pattern &p, const uint32_t *idx, Bind &b) {
    for (unsigned k = 0; k < p.n_vars; k++) b.var[k].cls = KC_NONE;
    for (int k = CL_MAX_VARS; k < NBIND; k++) b.var[k].cls = KC_NONE;
    for (unsigned t = 0; t < p.n_templates; t++) {
        const cl_hdr h = s.S.hdr[idx[t]];
        if (!match_inst(s, p.t[t], h, idx[t], b)) return false;
    }
    return connected(s, idx, p.n_templates);
}

/* head opcodes of one pattern table -> seed classes                          */
CLF void setup_classes(FS &s, unsigned table) {
    s.n_cls = 0;
    const cl_pattern_blob *pb = s.pb;
    for (unsigned pi = 0; pi < pb->n_patterns; pi++) {
        const cl_pattern &p = pb->p[pi];
        if (p.table != table) continue;
        for (unsigned t = 0; t < p.n_templates; t++) {
            bool seen = false;
            for (unsigned c = 0; c < s.n_cls; c++) seen |= s.cls_op[c] == p.t[t].op;
            if (!seen && s.n_cls < (unsigned)MAX_CLS) s.cls_op[s.n_cls++] = p.t[t].op;
        }
    }
}
CLD int class_of(const FS &s, uint16_t op) {
    for (unsigned c = 0; c < s.n_cls; c++) if (s.cls_op[c] == op) return (int)c;
    return -1;
}

/* FindSeeds (patterns.py:189-191): per head opcode, the block positions whose
 * base opcode fits, in order -- ballot/popc compaction per class.            */
template <class G> CLF uint32_t seed_scan(const G &g, FS &s, uint32_t lo, uint32_t n) {
    PROF(g, s, PF_SEED);
    GFOR(g, i, n) if (i < n) {
        const uint16_t op = s.S.hdr[lo + i].op;
        s.clsid[i] = (uint8_t)class_of(s, op);
    }
    g.sync();
    uint32_t total = 0;
    for (unsigned c = 0; c < s.n_cls; c++) {
        s.cls_off[c] = total;
        GFOR(g, i, n) {
            const bool f = i < n && s.clsid[i] == c;
            uint32_t cnt;
            const uint32_t off = g.flag_exscan(f, cnt);
            if (f) { s.cand[total + off] = i; s.cidx[i] = total + off - s.cls_off[c]; }
            total += cnt;
        }
    }
    s.cls_off[s.n_cls] = total;
    g.sync();
    return total;
}

/* append helper: ordered (ballot/popc) compaction of this iteration's hits   */
template <class G> CLD void append_match(const G &g, FS &s, uint32_t &nm, bool ok, unsigned pi, unsigned nt,
                                         const uint32_t *pos, unsigned long long r) {
    uint32_t cnt;
    const uint32_t off = g.flag_exscan(ok, cnt);
    if (ok && nm + off < s.cap.M) {
        MatchRec m;
        m.pat = (uint8_t)pi; m.n = (uint8_t)nt; m.state = MS_UNDECIDED; m.pad = 0;
        m.pos[0] = pos[0]; m.pos[1] = nt > 1 ? pos[1] : NONE32; m.pos[2] = nt > 2 ? pos[2] : NONE32;
        m.seq = (uint32_t)pi << 20 | (uint32_t)r;
        s.mt[nm + off] = m;
    }
    nm += cnt;
}

/* the candidate product of one pattern, literally (patterns.py:189-215): every
 * tuple of rank < budget in itertools.product order                          */
template <class G> CLF void match_product(const G &g, FS &s, uint32_t lo, unsigned pi, uint32_t &nm) {
    const cl_pattern &p = s.pb->p[pi];
    const unsigned nt = p.n_templates;
    uint32_t cn[3] = { 1, 1, 1 }, cb[3] = { 0, 0, 0 };
    for (unsigned t = 0; t < nt; t++) {
        const int c = class_of(s, p.t[t].op);
        cn[t] = s.cls_off[c + 1] - s.cls_off[c];
        cb[t] = s.cls_off[c];
        if (cn[t] == 0) return;
    }
    unsigned long long T = (unsigned long long)cn[0] * cn[1] * cn[2];
    if (T > s.pb->budget) T = s.pb->budget;                     /* :194-198 */
    const uint32_t Tl = (uint32_t)T;
    GFOR(g, r, Tl) {
        bool ok = false;
        uint32_t idx[3] = { NONE32, NONE32, NONE32 };
        if (r < Tl) {
            uint32_t q = r, i2 = 0, i1 = 0;
            if (nt > 2) { i2 = q % cn[2]; q /= cn[2]; }
            if (nt > 1) { i1 = q % cn[1]; q /= cn[1]; }
            idx[0] = s.cand[cb[0] + q];
            ok = true;
            if (nt > 1) { idx[1] = s.cand[cb[1] + i1]; ok = idx[0] < idx[1]; }
            if (nt > 2) { idx[2] = s.cand[cb[2] + i2]; ok = ok && idx[1] < idx[2]; }
            if (ok) {
                uint32_t abs_idx[3] = { lo + idx[0], lo + idx[1], lo + idx[2] };
                Bind b;
                ok = check_tuple(s, p, abs_idx, b);
            }
        }
        append_match(g, s, nm, ok, pi, nt, idx, r);
    }
}

/* match_patterns (patterns.py:181-216) of one block.
 * Join form: the work items are the (pattern, anchor seed) pairs of all
 * patterns, flattened so that lanes stay busy; every other instruction of a
 * tuple is the SSA definition of the operand that links it to an already
 * resolved one (unique), so the candidate product collapses to one tuple per
 * anchor.  The tuple's rank in itertools.product order still decides the
 * budget cut (G1) and the list order.  A link that is not an SSA value (RZ,
 * PT, an immediate...) sends its pattern to the literal product.            */
template <class G> CLF uint32_t match_block(const G &g, FS &s, uint32_t lo, uint32_t n, unsigned table) {
    PROF(g, s, PF_MATCH);
    if (seed_scan(g, s, lo, n) == 0) return 0;
    const cl_pattern_blob *pb = s.pb;
    uint32_t pref[CL_MAX_PATTERNS + 1];
    uint32_t product_mask = 0, items = 0;
    for (unsigned pi = 0; pi < pb->n_patterns; pi++) {
        const cl_pattern &p = pb->p[pi];
        pref[pi] = items;
        if (p.table != table) continue;
        bool empty = false;
        for (unsigned t = 0; t < p.n_templates; t++) {
            const int c = class_of(s, p.t[t].op);
            empty |= s.cls_off[c + 1] == s.cls_off[c];
        }
        if (empty) continue;
        if (!p.join_ok || s.odd_defs) { product_mask |= 1u << pi; continue; }
        const int ca = class_of(s, p.t[p.join_order[0]].op);
        items += s.cls_off[ca + 1] - s.cls_off[ca];
    }
    pref[pb->n_patterns] = items;
    uint32_t nm = 0, fb_mask = 0;
    GFOR(g, it, items) {
        bool ok = it < items;
        unsigned pi = 0, nt = 1;
        uint32_t idx[3] = { NONE32, NONE32, NONE32 }, pos[3] = { NONE32, NONE32, NONE32 };
        unsigned long long r = 0;
        if (ok) {
            while (pref[pi + 1] <= it) pi++;
            const cl_pattern &p = pb->p[pi];
            nt = p.n_templates;
            uint32_t cn[3] = { 1, 1, 1 };
            const unsigned ta = p.join_order[0];
            for (unsigned t = 0; t < nt; t++) { const int c = class_of(s, p.t[t].op); cn[t] = s.cls_off[c + 1] - s.cls_off[c]; }
            idx[ta] = lo + s.cand[s.cls_off[class_of(s, p.t[ta].op)] + (it - pref[pi])];
            for (unsigned k = 1; k < nt && ok; k++) {
                const unsigned t = p.join_order[k], from = p.join_from[k];
                const cl_hdr hf = s.S.hdr[idx[from]];
                const cl_template &tf = p.t[from];
                if (hf.n_defs != tf.n_defs || hf.n_aux != tf.n_aux || hf.n_uses != tf.n_uses || (hf.flags & CL_IF_EXT)) { ok = false; break; }
                const unsigned long long mm = s.ms[hf.modset].mask;
                if ((mm & tf.mods_all) != tf.mods_all || (mm & tf.mods_none)) { ok = false; break; }
                const opnd o = get_slot(s, hf, idx[from], has_guard(hf) + p.join_slot[k]);
                if (!is_value(o)) {
                    /* the link must equal a def operand of the missing instruction: with defs being
                     * values, RZ or predicates only (odd_defs == 0) nothing else can match        */
                    const unsigned ko = kind_of(o.tag);
                    if (ko == CL_K_RZ || ko == CL_K_URZ || ko == CL_K_PRED) fb_mask |= 1u << pi;
                    ok = false;
                    break;
                }
                const uint32_t dp = o.pay < s.cap.V ? s.defpos[o.pay] : NONE32;
                if (dp == NONE32 || dp < lo || dp >= lo + n || s.S.hdr[dp].op != p.t[t].op) { ok = false; break; }
                idx[t] = dp;
            }
            if (ok && nt > 1) ok = idx[0] < idx[1] && (nt < 3 || idx[1] < idx[2]);
            if (ok) {
                r = s.cidx[idx[0] - lo];
                if (nt > 1) r = r * cn[1] + s.cidx[idx[1] - lo];
                if (nt > 2) r = r * cn[2] + s.cidx[idx[2] - lo];
                ok = r < pb->budget;
            }
            if (ok) { Bind b; ok = check_tuple(s, p, idx, b); }
            for (unsigned t = 0; t < nt; t++) pos[t] = idx[t] - lo;
        }
        append_match(g, s, nm, ok, pi, nt, pos, r);
    }
    if (nm > s.cap.M) { fail(s, CL_ST_CAPACITY); g.sync(); return 0; }
    if (g.any(fb_mask != 0)) {
        /* rare: drop what the join found for those patterns and enumerate their product */
        uint32_t all = 0;
        for (unsigned pi = 0; pi < pb->n_patterns; pi++) if (g.any((fb_mask >> pi) & 1u)) all |= 1u << pi;
        g.sync();
        uint32_t kept = 0;
        const uint32_t have = nm < s.cap.M ? nm : s.cap.M;
        if (g.rank == 0) {
            for (uint32_t m = 0; m < have; m++) if (!((all >> s.mt[m].pat) & 1u)) s.mt[kept++] = s.mt[m];
        }
        nm = g.bcast0(kept);
        product_mask |= all;
        g.sync();
    }
    for (unsigned pi = 0; pi < pb->n_patterns; pi++)
        if ((product_mask >> pi) & 1u) match_product(g, s, lo, pi, nm);
    g.sync();
    if (nm > s.cap.M) { fail(s, CL_ST_CAPACITY); g.sync(); return 0; }
    return nm;
}

/* select_matches (patterns.py:241-252).  The stable sort key is
 * (start_pos, -len, list order); the greedy scan keeps a match iff no kept
 * match of smaller key overlaps it.  Parallel form: every round each
 * undecided match bids for its positions with its key (atomicMin); a match
 * that owns all of them has no smaller undecided rival and no kept rival, so
 * the sequential scan would keep it too; a match touching a kept position is
 * dropped.  Kept matches have distinct start positions, so ordered compaction
 * over positions yields them in sorted order.                               */
CLD unsigned long long match_key(const MatchRec &m) {
    return (unsigned long long)m.pos[0] << 32 | (unsigned long long)(3u - m.n) << 30 | (m.seq & 0x3FFFFFFFu);
}
template <class G> CLF uint32_t select_block(const G &g, FS &s, uint32_t n, uint32_t nm, uint32_t bi,
                                             uint32_t nsel) {
    PROF(g, s, PF_SELECT);
    GFOR(g, p, n) if (p < n) { s.keep[p] = 0; s.sel_at[p] = NONE32; }
    g.sync();
    for (;;) {
        GFOR(g, p, n) if (p < n && !s.keep[p]) s.owner[p] = NONE64;
        g.sync();
        GFOR(g, m, nm) if (m < nm && s.mt[m].state == MS_UNDECIDED) {
            MatchRec &r = s.mt[m];
            bool clash = false;
            for (unsigned t = 0; t < r.n; t++) clash |= s.keep[r.pos[t]] != 0;
            if (clash) r.state = MS_REJECTED;
            else for (unsigned t = 0; t < r.n; t++) p_min64(s, &s.owner[r.pos[t]], match_key(r));
        }
        g.sync();
        bool left = false;
        GFOR(g, m, nm) if (m < nm && s.mt[m].state == MS_UNDECIDED) {
            MatchRec &r = s.mt[m];
            const unsigned long long key = match_key(r);
            bool mine = true;
            for (unsigned t = 0; t < r.n; t++) mine &= s.owner[r.pos[t]] == key;
            if (mine) {
                r.state = MS_SELECTED;
                for (unsigned t = 0; t < r.n; t++) s.keep[r.pos[t]] = 1;
                s.sel_at[r.pos[0]] = m;
            } else
                left = true;
        }
        const bool again = g.any(left);
        g.sync();
        if (!again) break;
    }
    uint32_t count = 0;
    GFOR(g, p, n) {
        const bool f = p < n && s.sel_at[p] != NONE32;
        uint32_t cnt;
        const uint32_t off = g.flag_exscan(f, cnt);
        if (f && nsel + count + off < s.cap.S) {
            const MatchRec &m = s.mt[s.sel_at[p]];
            SelRec r;
            r.pat = m.pat; r.n = m.n; r.pad0 = r.pad1 = 0; r.blk = bi;
            r.pos[0] = m.pos[0]; r.pos[1] = m.pos[1]; r.pos[2] = m.pos[2];
            s.sel[nsel + count + off] = r;
        }
        count += cnt;
    }
    g.sync();
    if (nsel + count > s.cap.S) { fail(s, CL_ST_CAPACITY); g.sync(); return 0; }
    return count;
}

/* CL_EV_MATCH events of one block (match-only runs, emit_matches)            */
template <class G> CLF void emit_match_events(const G &g, FS &s, uint32_t seq, uint32_t nm, uint32_t sel0,
                                              uint32_t nsel) {
    GFOR(g, m, nm) if (m < nm) {
        const MatchRec &r = s.mt[m];
        push_event(s, seq, CL_EV_MATCH, r.seq, r.pat, r.pos[0], r.pos[1], r.pos[2]);
    }
    GFOR(g, j, nsel) if (j < nsel) {
        const SelRec &r = s.sel[sel0 + j];
        push_event(s, seq, CL_EV_MATCH, 0x80000000u | j, r.pat | 1u << 16, r.pos[0], r.pos[1], r.pos[2]);
    }
}

/* ------------------------------------------------------------------ rewrites */
/* One lane plans one selected match, once, into a staging record: new
 * instructions, values and immediates carry ids *relative* to the match
 * (CL_T_REL in the slot tag).  An exclusive scan over the block's matches in
 * select order then yields the id bases (vid, iid and immediate index are
 * allocated in exactly the reference's order, G3; refused rewrites keep what
 * they allocated before giving up, G4) and a fix-up pass writes the records
 * to their final place.                                                     */
static constexpr uint16_t CL_T_REL = 1u << 15;      /* payload is relative to the match's base */
static constexpr int ST_RECS = 6, ST_VALS = 4, ST_IMMS = 8, ST_UPD = 3, ST_DROP = 4;

struct SRec {                      /* a staged record: at most one def and three uses */
    uint16_t op, modset;
    uint8_t n_defs, n_uses, iid, pad;
    uint16_t tag[4];
    uint32_t pay[4];
};
struct Stage {
    SRec rec[ST_RECS];
    cl_imm imm[ST_IMMS];
    uint32_t upd_vid[ST_UPD];      /* existing values redefined ...                */
    uint32_t drop_vid[ST_DROP];
    int8_t val_def[ST_VALS];       /* relative iid of the defining record, -1 none */
    uint8_t upd_iid[ST_UPD];       /* ... by the record with this relative iid     */
    uint8_t ok, rm, nins, retag, nv, nq, nupd, ndrop, ni;
    uint32_t vbase, ibase, mbase;  /* after the scan                               */
};

struct RW {
    FS *s;
    Stage *st;
    uint32_t idx[3];               /* stream positions of the matched records      */
    cl_hdr h[3];
    unsigned n, pat;
    bool overflow;
    uint32_t *stw;                 /* status word of the function that owns the match */
};

CLD opnd rw_value(RW &c, uint32_t origin) {               /* LiftedFunction.new_value */
    Stage &st = *c.st;
    opnd o; o.tag = (uint16_t)(CL_K_VALUE | CL_T_REL); o.pay = st.nv;
    (void)origin;                  /* always "pair" in this pass (patterns.py:292,356,405) */
    if (st.nv < ST_VALS) { st.val_def[st.nv] = -1; st.nv++; } else c.overflow = true;
    return o;
}
CLD opnd rw_imm(RW &c, unsigned long long bits, unsigned long long text, bool hextext) {
    Stage &st = *c.st;
    opnd o; o.tag = (uint16_t)(CL_K_IMM | CL_T_REL | (hextext ? CL_T_IMM_HEXTEXT : 0)); o.pay = st.nq;
    if (st.nq < ST_IMMS) { st.imm[st.nq].bits = bits; st.imm[st.nq].text = text; st.nq++; } else c.overflow = true;
    return o;
}
/* bits/text of an immediate operand, staged or already in the function's table */
CLD cl_imm rw_imm_of(const RW &c, opnd o) {
    return (o.tag & CL_T_REL) ? c.st->imm[o.pay & (ST_IMMS - 1)] : c.s->imm[o.pay];
}
/* LiftedFunction.make_inst (ssir.py:237-241); iid relative                    */
CLD Rec rw_make(RW &c, uint16_t op, uint16_t modset, const opnd *defs, unsigned nd, const opnd *uses,
                unsigned nu) {
    Rec r;
    r.h.iid = c.st->ni++;
    r.h.op = op; r.h.modset = modset;
    r.h.n_defs = (uint8_t)nd; r.h.n_aux = 0; r.h.n_uses = (uint8_t)nu; r.h.flags = 0; r.h.ext = 0;
    unsigned k = 0;
    for (unsigned i = 0; i < nd; i++, k++) { r.tag[k] = defs[i].tag; r.pay[k] = defs[i].pay; }
    for (unsigned i = 0; i < nu; i++, k++) { r.tag[k] = uses[i].tag; r.pay[k] = uses[i].pay; }
    for (; k < 8; k++) { r.tag[k] = 0; r.pay[k] = 0; }
    return r;
}
CLD void rw_push(RW &c, const Rec &r) {
    Stage &st = *c.st;
    if (st.nins < ST_RECS && (unsigned)r.h.n_defs + r.h.n_uses <= 4) {
        SRec &q = st.rec[st.nins++];
        q.op = r.h.op; q.modset = r.h.modset; q.n_defs = r.h.n_defs; q.n_uses = r.h.n_uses; q.iid = (uint8_t)r.h.iid; q.pad = 0;
        for (unsigned k = 0; k < 4; k++) { q.tag[k] = r.tag[k]; q.pay[k] = r.pay[k]; }
    } else c.overflow = true;
}
/* info.def_iid = inst.iid for a staged (relative) or an existing value        */
CLD void rw_set_def_iid(RW &c, opnd v, uint32_t iid_rel) {
    Stage &st = *c.st;
    if (v.tag & CL_T_REL) { if (v.pay < (uint32_t)ST_VALS) st.val_def[v.pay] = (int8_t)iid_rel; }
    else if (st.nupd < ST_UPD) { st.upd_vid[st.nupd] = v.pay; st.upd_iid[st.nupd] = (uint8_t)iid_rel; st.nupd++; }
    else c.overflow = true;
}
CLD void rw_drop(RW &c, opnd o) {                       /* _drop_values :314-317 */
    Stage &st = *c.st;
    if (!is_value(o)) return;
    if (st.ndrop < ST_DROP) st.drop_vid[st.ndrop++] = o.pay; else c.overflow = true;
}
CLD void rw_fail(RW &c, uint32_t code) { if (c.s->solo) { if (!*c.stw) *c.stw = code; } else a_cas0(c.stw, code); }

/* _escapes (patterns.py:259-263) against the def-use snapshot of the block:
 * a value escapes iff it has more use sites than the group itself holds.    */
CLF bool rw_escapes(RW &c, uint32_t vid) {
    FS &s = *c.s;
    uint32_t inside = 0;
    for (unsigned t = 0; t < c.n; t++)
        for_value_operands(s, c.h[t], c.idx[t], [&](uint32_t v) { inside += v == vid; });
    return vid < s.cap.V && s.usecnt[vid] != inside;
}
/* _safe (patterns.py:266-275)                                                 */
CLF bool rw_safe(RW &c, const opnd *redef, unsigned nredef) {
    FS &s = *c.s;
    for (unsigned t = 0; t < c.n; t++) {
        const unsigned d0 = def0(c.h[t]), nd = (unsigned)c.h[t].n_defs + c.h[t].n_aux;
        for (unsigned k = 0; k < nd; k++) {
            opnd d = get_slot(s, c.h[t], c.idx[t], d0 + k);
            if (!is_value(d)) continue;
            bool re = false;
            for (unsigned j = 0; j < nredef; j++) re |= is_value(redef[j]) && redef[j].pay == d.pay;
            if (!re && rw_escapes(c, d.pay)) return false;
        }
    }
    return true;
}
/* _pack_pair (patterns.py:278-300); CL_K_NONE stands for None                 */
CLF opnd rw_pack_pair(RW &c, opnd lo, opnd hi) {
    const bool lo_zero = is_zero(lo), hi_zero = is_zero(hi);
    opnd none; none.tag = CL_K_NONE; none.pay = 0;
    if (lo_zero && hi_zero) return none;
    if (is_imm(lo) && hi_zero) {
        const cl_imm im = rw_imm_of(c, lo);
        return rw_imm(c, im.bits & 0xFFFFFFFFull, im.text, (lo.tag & CL_T_IMM_HEXTEXT) != 0);
    }
    if (is_imm(lo) && is_imm(hi)) {
        const unsigned long long bits = (rw_imm_of(c, lo).bits & 0xFFFFFFFFull) | (rw_imm_of(c, hi).bits & 0xFFFFFFFFull) << 32;
        return rw_imm(c, bits, bits, true);
    }
    if (lo_zero && is_imm(hi)) {
        const unsigned long long bits = (rw_imm_of(c, hi).bits & 0xFFFFFFFFull) << 32;
        return rw_imm(c, bits, bits, true);
    }
    opnd d = rw_value(c, CL_ORG_PAIR);
    opnd u[2];
    u[0] = lo_zero ? rw_imm(c, 0, 0, true) : strip(lo);
    u[1] = hi_zero ? rw_imm(c, 0, 0, true) : strip(hi);
    Rec pk = rw_make(c, CL_OP_PACK64, CL_MS_NONE, &d, 1, u, 2);
    rw_set_def_iid(c, d, pk.h.iid);
    rw_push(c, pk);
    return d;
}
/* _unpack_into (patterns.py:303-311)                                          */
CLF void rw_unpack_into(RW &c, opnd src, opnd lo_ref, opnd hi_ref) {
    opnd refs[2] = { lo_ref, hi_ref };
    for (int k = 0; k < 2; k++) {
        if (!is_value(refs[k])) continue;
        opnd d = value_ref(refs[k].pay);
        Rec up = rw_make(c, CL_OP_UNPACK64, k ? CL_MS_HI : CL_MS_LO, &d, 1, &src, 1);
        if (!(d.pay < c.s->cap.V && c.s->alive[d.pay])) { rw_fail(c, CL_ST_KEY_ERROR); return; }
        rw_set_def_iid(c, d, up.h.iid);
        rw_push(c, up);
    }
}
CLD bool rw_redefine(RW &c, opnd res, uint32_t iid) {
    if (!is_value(res)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
    if (!(res.pay < c.s->cap.V && c.s->alive[res.pay])) { rw_fail(c, CL_ST_KEY_ERROR); return false; }
    rw_set_def_iid(c, value_ref(res.pay), iid);
    return true;
}

/* _rw_iadd364 (patterns.py:324-362)                                           */
CLF bool rw_iadd364(RW &c) {
    FS &s = *c.s;
    const cl_hdr &lo = c.h[0], &hi = c.h[1];
    opnd carry = get_aux(s, lo, c.idx[0], 0);
    opnd redef[2] = { get_def(s, lo, c.idx[0], 0), get_def(s, hi, c.idx[1], 0) };
    if (!rw_safe(c, redef, 2)) return false;
    opnd ops[3];
    unsigned nops = 0;
    for (unsigned k = 0; k < 3; k++) {
        opnd lo_op = get_use(s, lo, c.idx[0], k), hi_op = get_use(s, hi, c.idx[1], k);
        const bool neg_lo = o_neg(lo_op), not_hi = o_not(hi_op);
        const bool plain = !neg_lo && !not_hi && !o_not(lo_op) && !o_neg(hi_op);
        if (plain) {
            opnd p = rw_pack_pair(c, lo_op, hi_op);
            if (!is_none(p)) ops[nops++] = p;
        } else if (neg_lo && not_hi) {
            opnd p = rw_pack_pair(c, strip(lo_op), strip(hi_op));
            if (is_none(p)) return false;
            if (is_imm(p)) {                       /* Imm(-p.int_value(64) & M64, p.text) :348 */
                const cl_imm im = rw_imm_of(c, p);
                ops[nops++] = rw_imm(c, 0ull - im.bits, im.text, (p.tag & CL_T_IMM_HEXTEXT) != 0);
            } else {
                p.tag |= CL_T_NEG;
                ops[nops++] = p;
            }
        } else
            return false;                          /* mixed negation :353 */
    }
    if (!nops) return false;
    opnd d = rw_value(c, CL_ORG_PAIR);
    Rec agg = rw_make(c, CL_OP_IADD364, CL_MS_NONE, &d, 1, ops, nops);
    rw_set_def_iid(c, d, agg.h.iid);
    rw_push(c, agg);
    rw_unpack_into(c, d, redef[0], redef[1]);
    rw_drop(c, carry);
    c.st->rm = 3;
    return true;
}
/* "mod:<var>" binding of _match_opcode (patterns.py:163-166) for the matched
 * instruction t: first modifier of its tuple that belongs to the choice group */
CLD unsigned rw_modvar(const RW &c, unsigned t, unsigned modvar) {
    const cl_template &tm = c.s->pb->p[c.pat].t[t];
    for (unsigned k = 0; k < tm.n_modvars; k++)
        if (tm.modvar_var[k] == modvar) return c.s->ms[c.h[t].modset].first[tm.modvar_group[k]];
    return 0;
}
/* _rw_isetp64 (patterns.py:371-390)                                           */
CLF bool rw_isetp64(RW &c) {
    FS &s = *c.s;
    const cl_pattern &p = s.pb->p[c.pat];
    const cl_hdr &lo = c.h[0], &hi = c.h[1];
    opnd res = get_def(s, hi, c.idx[1], 0);
    if (!rw_safe(c, &res, 1)) return false;
    const unsigned cond = s.pb->group_pos[rw_modvar(c, 0, p.modvar_cond) & 63];
    const unsigned bop = s.pb->group_pos[rw_modvar(c, 0, p.modvar_bop) & 63];
    const unsigned unsigned_hi = has_mod(s, hi, CL_MB_U32);
    opnd u[3];
    u[0] = rw_pack_pair(c, get_use(s, lo, c.idx[0], 0), get_use(s, hi, c.idx[1], 0));
    u[1] = rw_pack_pair(c, get_use(s, lo, c.idx[0], 1), get_use(s, hi, c.idx[1], 1));
    if (is_none(u[0])) u[0] = rw_imm(c, 0, 0, true);
    if (is_none(u[1])) u[1] = rw_imm(c, 0, 0, true);
    u[2] = get_use(s, hi, c.idx[1], 2);
    if (!is_value(res)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
    opnd d = value_ref(res.pay);
    Rec agg = rw_make(c, CL_OP_ISETP64, s.pb->isetp64_ms[cond & 7][unsigned_hi][bop & 7], &d, 1, u, 3);
    if (!rw_redefine(c, res, agg.h.iid)) return false;
    rw_push(c, agg);
    rw_drop(c, get_def(s, lo, c.idx[0], 0));
    c.st->rm = 3;
    return true;
}
/* _rw_lea64 (patterns.py:393-411)                                             */
CLF bool rw_lea64(RW &c) {
    FS &s = *c.s;
    const cl_hdr &lo = c.h[0], &hi = c.h[1];
    opnd carry = get_aux(s, lo, c.idx[0], 0);
    opnd redef[2] = { get_def(s, lo, c.idx[0], 0), get_def(s, hi, c.idx[1], 0) };
    if (!rw_safe(c, redef, 2)) return false;
    opnd a64 = rw_pack_pair(c, get_use(s, lo, c.idx[0], 0), get_use(s, hi, c.idx[1], 2));
    opnd b64 = rw_pack_pair(c, get_use(s, lo, c.idx[0], 1), get_use(s, hi, c.idx[1], 1));
    if (is_none(a64) || is_none(b64)) return false;
    opnd d = rw_value(c, CL_ORG_PAIR), u[3] = { b64, a64, get_use(s, lo, c.idx[0], 2) };
    Rec agg = rw_make(c, CL_OP_LEA64, CL_MS_NONE, &d, 1, u, 3);
    rw_set_def_iid(c, d, agg.h.iid);
    rw_push(c, agg);
    rw_unpack_into(c, d, redef[0], redef[1]);
    rw_drop(c, carry);
    c.st->rm = 3;
    return true;
}
/* _rw_imad_wide (patterns.py:414-418): in-place retag, applied by the fix-up  */
CLF bool rw_imad_wide(RW &c) {
    c.st->retag = 1;
    return true;
}
/* tail of mov64 / cast64 / shl64 / shr64 (patterns.py:433-439 and alike)      */
CLF bool rw_finish_pack(RW &c, const Rec &agg, unsigned n_feed) {
    FS &s = *c.s;
    rw_push(c, agg);
    c.st->rm = (uint8_t)(1u << n_feed);
    for (unsigned t = 0; t < n_feed; t++) {
        opnd d = get_def(s, c.h[t], c.idx[t], 0);
        if (!is_value(d)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
        if (!rw_escapes(c, d.pay)) { rw_drop(c, d); c.st->rm |= (uint8_t)(1u << t); }
    }
    return true;
}
/* _rw_mov64 (patterns.py:421-439)                                             */
CLF bool rw_mov64(RW &c) {
    FS &s = *c.s;
    opnd clo = get_use(s, c.h[0], c.idx[0], 0), chi = get_use(s, c.h[1], c.idx[1], 0);
    if (kind_of(clo.tag) != CL_K_CONSTMEM || kind_of(chi.tag) != CL_K_CONSTMEM) return false;
    const uint32_t mask = (1u << CL_CM_OFFSET_BITS) - 1u;
    if ((clo.pay >> CL_CM_OFFSET_BITS) != (chi.pay >> CL_CM_OFFSET_BITS) ||
        (chi.pay & mask) != (clo.pay & mask) + 4u) return false;
    opnd res = get_def(s, c.h[2], c.idx[2], 0);
    if (!is_value(res)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
    opnd d = value_ref(res.pay), u;
    u.tag = (uint16_t)(CL_K_CONSTMEM | 2u << CL_T_WIDTH_SHIFT); u.pay = clo.pay;
    Rec agg = rw_make(c, CL_OP_MOV64, CL_MS_NONE, &d, 1, &u, 1);
    if (!rw_redefine(c, res, agg.h.iid)) return false;
    return rw_finish_pack(c, agg, 2);
}
/* _rw_cast64 (patterns.py:442-453)                                            */
CLF bool rw_cast64(RW &c) {
    FS &s = *c.s;
    opnd res = get_def(s, c.h[1], c.idx[1], 0);
    if (!is_value(res)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
    opnd d = value_ref(res.pay), u = strip(get_use(s, c.h[1], c.idx[1], 0));
    Rec agg = rw_make(c, CL_OP_CAST64, CL_MS_NONE, &d, 1, &u, 1);
    if (!rw_redefine(c, res, agg.h.iid)) return false;
    return rw_finish_pack(c, agg, 1);
}
/* _rw_shl64 / _rw_shr64 (patterns.py:456-495)                                 */
CLF bool rw_shift64(RW &c, bool right) {
    FS &s = *c.s;
    const bool is_signed = has_mod(s, c.h[0], CL_MB_S32);
    opnd src = right ? rw_pack_pair(c, get_use(s, c.h[1], c.idx[1], 0), get_use(s, c.h[0], c.idx[0], 2))
                     : rw_pack_pair(c, get_use(s, c.h[0], c.idx[0], 0), get_use(s, c.h[0], c.idx[0], 2));
    if (is_none(src)) return false;
    opnd res = get_def(s, c.h[2], c.idx[2], 0);
    if (!is_value(res)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
    opnd d = value_ref(res.pay), u[2] = { src, get_use(s, c.h[0], c.idx[0], 1) };
    Rec agg = rw_make(c, right ? CL_OP_SHR64 : CL_OP_SHL64,
                      right ? (is_signed ? CL_MS_S64 : CL_MS_U64) : CL_MS_NONE, &d, 1, u, 2);
    if (!rw_redefine(c, res, agg.h.iid)) return false;
    return rw_finish_pack(c, agg, 2);
}
/* Binding of a pattern variable = key of the first slot (template order, then
 * defs/aux/uses) that mentions it -- what Bindings.vars holds after a
 * successful unification.  Then _var_operand (patterns.py:514-524).           */
CLF bool rw_var_operand(RW &c, unsigned var, opnd *out) {
    FS &s = *c.s;
    const cl_pattern &p = s.pb->p[c.pat];
    for (unsigned t = 0; t < c.n; t++) {
        const cl_template &tm = p.t[t];
        const unsigned ns = (unsigned)tm.n_defs + tm.n_aux + tm.n_uses;
        for (unsigned k = 0; k < ns; k++) {
            if (tm.slot[k].kind != CL_S_VAR || tm.slot[k].var != var) continue;
            const okey key = operand_key(s, get_slot(s, c.h[t], c.idx[t], has_guard(c.h[t]) + k));
            switch (key.cls) {
            case KC_V: *out = value_ref((uint32_t)key.v); return true;
            case KC_IMM: *out = rw_imm(c, key.v, key.v, true); return true;
            case KC_CM: out->tag = (uint16_t)(CL_K_CONSTMEM | 1u << CL_T_WIDTH_SHIFT); out->pay = (uint32_t)key.v; return true;
            case KC_RZ: out->tag = CL_K_RZ; out->pay = 0; return true;
            default: rw_fail(c, CL_ST_ASSERTION_ERROR); return false;
            }
        }
    }
    rw_fail(c, CL_ST_KEY_ERROR);
    return false;
}
/* _rw_xmad (patterns.py:498-511)                                              */
CLF bool rw_xmad(RW &c) {
    FS &s = *c.s;
    const cl_pattern &p = s.pb->p[c.pat];
    opnd dres = get_def(s, c.h[2], c.idx[2], 0);
    if (!rw_safe(c, &dres, 1)) return false;
    opnd u[3];
    if (!rw_var_operand(c, p.var_a, &u[0])) return false;
    if (!rw_var_operand(c, p.var_b, &u[1])) return false;
    if (!rw_var_operand(c, p.var_c, &u[2])) return false;
    if (!is_value(dres)) { rw_fail(c, CL_ST_ATTRIBUTE_ERROR); return false; }
    opnd d = value_ref(dres.pay);
    Rec agg = rw_make(c, CL_OP_IMAD, CL_MS_NONE, &d, 1, u, 3);
    if (!rw_redefine(c, dres, agg.h.iid)) return false;
    rw_push(c, agg);
    for (unsigned t = 0; t < 2; t++)
        for (unsigned k = 0; k < c.h[t].n_defs; k++) rw_drop(c, get_def(s, c.h[t], c.idx[t], k));
    c.st->rm = 7;
    return true;
}
CLF bool run_rewrite(RW &c) {
    switch (c.s->pb->p[c.pat].rewrite) {
    case CL_RW_IADD364: return rw_iadd364(c);
    case CL_RW_ISETP64: return rw_isetp64(c);
    case CL_RW_LEA64: return rw_lea64(c);
    case CL_RW_IMAD_WIDE: return rw_imad_wide(c);
    case CL_RW_MOV64: return rw_mov64(c);
    case CL_RW_CAST64: return rw_cast64(c);
    case CL_RW_SHL64: return rw_shift64(c, false);
    case CL_RW_SHR64: return rw_shift64(c, true);
    case CL_RW_XMAD: return rw_xmad(c);
    }
    rw_fail(c, CL_ST_UNSUPPORTED);
    return false;
}

/* fix-up of one staged match once the bases are known                        */
CLF void apply_stage(FS &s, const SelRec &m, Stage &st, uint32_t lo, uint32_t out) {
    for (unsigned k = 0; k < st.nv; k++) {
        const uint32_t v = st.vbase + k;
        if (v >= s.cap.V) continue;
        s.alive[v] = 1; s.origin[v] = CL_ORG_PAIR;
        s.def_iid[v] = st.val_def[k] < 0 ? -1 : (int32_t)(st.ibase + (uint32_t)st.val_def[k]);
        s.usecnt[v] = 0; s.defpos[v] = NONE32;
    }
    for (unsigned k = 0; k < st.nq; k++) if (st.mbase + k < s.cap.Q) s.imm[st.mbase + k] = st.imm[k];
    if (!st.ok) return;                      /* refused: the allocations above leak (G4) */
    for (unsigned r = 0; r < st.nins; r++) {
        const SRec q = st.rec[r];
        Rec rec;
        rec.h.iid = st.ibase + q.iid; rec.h.op = q.op; rec.h.modset = q.modset;
        rec.h.n_defs = q.n_defs; rec.h.n_aux = 0; rec.h.n_uses = q.n_uses; rec.h.flags = 0; rec.h.ext = 0;
        for (unsigned k = 0; k < 8; k++) { rec.tag[k] = k < 4 ? q.tag[k] : 0; rec.pay[k] = k < 4 ? q.pay[k] : 0; }
        const unsigned ns = (unsigned)rec.h.n_defs + rec.h.n_uses;
        for (unsigned k = 0; k < ns; k++) {
            if (rec.tag[k] & CL_T_REL) {
                rec.pay[k] += kind_of(rec.tag[k]) == CL_K_VALUE ? st.vbase : st.mbase;
                rec.tag[k] &= (uint16_t)~CL_T_REL;
            }
            if (k < rec.h.n_defs) continue;
            if (kind_of(rec.tag[k]) == CL_K_VALUE) { if (rec.pay[k] < s.cap.V) p_add(s, &s.usecnt[rec.pay[k]], 1u); }
            else if (kind_of(rec.tag[k]) == CL_K_MEMREF) {
                const cl_memref &mr = s.mem[rec.pay[k]];
                if (kind_of(mr.base_tag) == CL_K_VALUE) p_add(s, &s.usecnt[mr.base_pay], 1u);
                if (kind_of(mr.ureg_tag) == CL_K_VALUE) p_add(s, &s.usecnt[mr.ureg_pay], 1u);
            }
        }
        st_rec(s, out + r, rec);
    }
    for (unsigned k = 0; k < st.nupd; k++) if (st.upd_vid[k] < s.cap.V) s.def_iid[st.upd_vid[k]] = (int32_t)(st.ibase + st.upd_iid[k]);
    for (unsigned k = 0; k < st.ndrop; k++) if (st.drop_vid[k] < s.cap.V) s.alive[st.drop_vid[k]] = 0;
    if (st.retag) {                          /* _rw_imad_wide :414-418 */
        cl_hdr &h = s.S.hdr[lo + m.pos[0]];
        h.modset = s.ms[h.modset].minus_wide;
        h.op = CL_OP_IMAD64;
    }
}

/* _apply_patterns (patterns.py:671-707): one round over all blocks.
 * Phase 1 matches and selects every block (matching never looks outside its
 * block); if nothing was selected the round is over.  Phase 2 walks the
 * blocks in order -- the escape test of block b must see the use counts left
 * by the rewrites of blocks < b (G5) -- compacting the stream from the right
 * end of the gap buffer to the left.                                        */
/* phase A: seed classes, def positions for the join, use counts for the escapes */
template <class G> CLF void ap_prepare(const G &g, FS &s, unsigned table) {
    setup_classes(s, table);
    build_usecount(g, s);
}
/* phase B: match + select every block; returns the number of selected matches */
template <class G> CLF uint32_t ap_match(const G &g, FS &s, unsigned table, uint32_t phase) {
    uint32_t nsel = 0;
    for (uint32_t bi = 0; bi < s.nb; bi++) {
        const uint32_t lo = s.bo[bi], n = s.bo[bi + 1] - lo;
        if (g.rank == 0) s.blk_sel[bi] = nsel;
        if (n == 0) continue;
        const uint32_t nm = match_block(g, s, lo, n, table);
        if (status(s)) return 0;
        if (nm == 0) continue;
        const uint32_t ns = select_block(g, s, n, nm, bi, nsel);
        if (status(s)) return 0;
        if (g.rank == 0) {
            for (uint32_t m = 0; m < nm; m++) s.st_matches[s.mt[m].pat]++;
            for (uint32_t j = 0; j < ns; j++) s.st_selected[s.sel[nsel + j].pat]++;
        }
        if (s.emit_matches) emit_match_events(g, s, phase << 28 | bi, nm, nsel, ns);
        nsel += ns;
        g.sync();
    }
    if (g.rank == 0) s.blk_sel[s.nb] = nsel;
    g.sync();
    return nsel;
}
/* phase C: plan, scan, emit block by block; returns the number of successful rewrites */
template <class G> CLF uint32_t ap_rewrite(const G &g, FS &s, uint32_t phase) {
    const uint32_t shift = s.cap.I - s.n;                    /* right-align the stream */
    move_recs(g, s, shift, 0, s.n);
    uint32_t wr = 0, total_ok = 0;
    for (uint32_t bi = 0; bi < s.nb; bi++) {
        const uint32_t lo = s.bo[bi] + shift, n = s.bo[bi + 1] - s.bo[bi];
        const uint32_t j0 = s.blk_sel[bi], ns = s.blk_sel[bi + 1] - j0;
        if (g.rank == 0) s.bo2[bi] = wr;
        if (ns == 0) {
            move_recs(g, s, wr, lo, n);
            wr += n;
            continue;
        }
        PROF(g, s, PF_PLAN);
        GFOR(g, p, n) if (p < n) { s.keep[p] = 1; s.inscnt[p] = 0; }
        g.sync();
        /* plan: one lane per match, once */
        bool over = false;
        GFOR(g, j, ns) if (j < ns) {
            const SelRec m = s.sel[j0 + j];
            Stage &st = s.stage[j0 + j];
            st.ok = st.rm = st.nins = st.retag = st.nv = st.nq = st.nupd = st.ndrop = 0;
            st.ni = 0;
            RW c;
            c.s = &s; c.st = &st; c.n = m.n; c.pat = m.pat; c.overflow = false; c.stw = s.st;
            for (unsigned t = 0; t < m.n; t++) { c.idx[t] = lo + m.pos[t]; c.h[t] = s.S.hdr[c.idx[t]]; }
            for (unsigned t = m.n; t < 3; t++) c.idx[t] = NONE32;
            st.ok = run_rewrite(c);
            over |= c.overflow;
        }
        if (g.any(over)) fail(s, CL_ST_UNSUPPORTED);
        g.sync();
        if (status(s)) return 0;
        /* exclusive scans in select order: id bases (G3) */
        uint32_t vb = s.next_vid, ib = s.next_iid, mb = s.n_imm, okc = 0;
        GFOR(g, j, ns) {
            uint32_t nv = 0, ni = 0, nq = 0, ok = 0;
            if (j < ns) { const Stage &st = s.stage[j0 + j]; nv = st.nv; ni = st.ni; nq = st.nq; ok = st.ok; }
            uint32_t tv, ti, tq, to;
            const uint32_t ov = g.exscan(nv, tv), oi = g.exscan(ni, ti), oq = g.exscan(nq, tq);
            g.exscan(ok, to);
            if (j < ns) {
                Stage &st = s.stage[j0 + j];
                st.vbase = vb + ov; st.ibase = ib + oi; st.mbase = mb + oq;
                const SelRec &m = s.sel[j0 + j];
                if (st.ok) {
                    s.inscnt[m.pos[m.n - 1]] = st.nins;                  /* anchor :689 */
                    for (unsigned t = 0; t < m.n; t++) if (st.rm >> t & 1) s.keep[m.pos[t]] = 0;
                }
            }
            vb += tv; ib += ti; mb += tq; okc += to;
        }
        if (vb > s.cap.V || mb > s.cap.Q) { fail(s, CL_ST_CAPACITY); g.sync(); return 0; }
        g.sync();
        /* output offsets of the block */
        uint32_t tot = 0;
        GFOR(g, p, n) {
            const uint32_t x = p < n ? (uint32_t)s.keep[p] + s.inscnt[p] : 0u;
            uint32_t t;
            const uint32_t o = g.exscan(x, t);
            if (p < n) s.outpos[p] = tot + o;
            tot += t;
        }
        if (wr + tot > lo) { fail(s, CL_ST_CAPACITY); g.sync(); return 0; }     /* gap exhausted */
        g.sync();
        /* fix-up: staged records to their place, value table, immediates */
        GFOR(g, j, ns) if (j < ns) {
            const SelRec m = s.sel[j0 + j];
            Stage &st = s.stage[j0 + j];
            apply_stage(s, m, st, lo, wr + s.outpos[m.pos[m.n - 1]]);
            if (!st.ok) push_event(s, phase << 28 | bi, CL_EV_REFUSED, j, m.pat, s.blk[bi].bid, 0, 0);
        }
        if (g.rank == 0)
            for (uint32_t j = 0; j < ns; j++) {
                const unsigned pat = s.sel[j0 + j].pat;
                if (s.stage[j0 + j].ok) s.st_rewrites[pat]++; else s.st_refused[pat]++;
            }
        g.sync();
        /* kept records move left; removed ones give their uses back */
        GFOR(g, p, n) if (p < n) {
            if (s.keep[p]) {
                Rec r;
                ld_rec(s, lo + p, r);
                st_rec(s, wr + s.outpos[p] + s.inscnt[p], r);
            } else {
                const cl_hdr h = s.S.hdr[lo + p];
                for_value_operands(s, h, lo + p, [&](uint32_t v) { if (v < s.cap.V) p_sub(s, &s.usecnt[v], 1u); });
            }
        }
        g.sync();
        wr += tot;
        s.next_vid = vb; s.next_iid = ib; s.n_imm = mb;
        total_ok += okc;
    }
    if (g.rank == 0) s.bo2[s.nb] = wr;
    { uint32_t *t = s.bo; s.bo = s.bo2; s.bo2 = t; }
    s.n = wr;
    g.sync();
    return total_ok;
}
template <class G> CLF uint32_t apply_patterns(const G &g, FS &s, unsigned table, uint32_t phase) {
    ap_prepare(g, s, table);
    const uint32_t nsel = ap_match(g, s, table, phase);
    if (status(s) || nsel == 0) return 0;
    return ap_rewrite(g, s, phase);
}

/* ordered in-place compaction of the stream by keep[] (block offsets follow) */
template <class G> CLF void compact_stream(const G &g, FS &s) {
    /* new offset of every block = kept records before its old start */
    uint32_t run = 0;
    uint32_t bi = 0;
    /* outpos[i] = kept before i */
    GFOR(g, i, s.n) {
        const uint32_t x = i < s.n ? (uint32_t)s.keep[i] : 0u;
        uint32_t t;
        const uint32_t o = g.exscan(x, t);
        if (i < s.n) s.outpos[i] = run + o;
        run += t;
    }
    (void)bi;
    g.sync();
    GFOR(g, b, s.nb + 1) if (b <= s.nb) {
        const uint32_t old = s.bo[b];
        s.bo2[b] = old < s.n ? s.outpos[old] : run;
    }
    g.sync();
    const uint32_t chunks = (s.n + g.size - 1) / g.size;
    for (uint32_t c = 0; c < chunks; c++) {
        const uint32_t i = c * g.size + g.rank;
        Rec r;
        const bool k = i < s.n && s.keep[i];
        uint32_t dst = 0;
        if (k) { ld_rec(s, i, r); dst = s.outpos[i]; }
        g.sync();
        if (k) st_rec(s, dst, r);
        g.sync();
    }
    { uint32_t *t = s.bo; s.bo = s.bo2; s.bo2 = t; }
    s.n = run;
}

/* remove_dead_pseudo (patterns.py:771-791).  The reference removes, round by
 * round, every pure instruction whose values have no users; the union of the
 * rounds is the least fixpoint of "dead", which chaotic iteration reaches in
 * any order, so dead marks and use-count decrements are applied on the fly. */
template <class G> CLF uint32_t remove_dead_pseudo(const G &g, FS &s) {
    PROF(g, s, PF_DCE);
    build_usecount(g, s);
    GFOR(g, i, s.n) if (i < s.n) s.keep[i] = 1;
    g.sync();
    uint32_t removed = 0;
    for (;;) {
        uint32_t mine = 0;
        GFOR(g, i, s.n) if (i < s.n && s.keep[i]) {
            const cl_hdr h = s.S.hdr[i];
            if (h.op >= CL_OP__COUNT || !(s.opflags[h.op] & CL_OPF_PURE)) continue;
            unsigned nd = 0; bool used = false;
            for_value_defs(s, h, i, [&](uint32_t v) { nd++; used |= v < s.cap.V && *(volatile uint32_t *)&s.usecnt[v] != 0; });
            if (!nd || used) continue;
            s.keep[i] = 0;
            mine++;
            for_value_defs(s, h, i, [&](uint32_t v) { if (v < s.cap.V) s.alive[v] = 0; });
            for_value_operands(s, h, i, [&](uint32_t v) { if (v < s.cap.V) p_sub(s, &s.usecnt[v], 1u); });
        }
        const uint32_t dead = g.sum(mine);
        g.sync();
        if (!dead) break;
        removed += dead;
    }
    if (removed) compact_stream(g, s);
    return removed;
}

/* simplify_packs + _redirect_values (patterns.py:710-764)                     */
CLD uint32_t final_of(const FS &s, uint32_t v) {
    while (v < s.cap.V && s.redirect[v] != NONE32) v = s.redirect[v];
    return v;
}
template <class G> CLF uint32_t simplify_packs(const G &g, FS &s, bool with_dce = true) {
    PROF(g, s, PF_SIMPLIFY);
    build_usecount(g, s);
    GFOR(g, v, s.next_vid) if (v < s.next_vid) s.redirect[v] = NONE32;
    g.sync();
    uint32_t mine = 0;
    GFOR(g, i, s.n) if (i < s.n) {
        const cl_hdr h = s.S.hdr[i];
        if (h.op != CL_OP_PACK64 || h.n_uses != 2) continue;
        opnd lo = get_use(s, h, i, 0), hi = get_use(s, h, i, 1);
        if (!is_value(lo) || !is_value(hi)) continue;
        if ((lo.tag | hi.tag) & (CL_T_NEG | CL_T_NOT)) continue;
        if (lo.pay >= s.cap.V || hi.pay >= s.cap.V) continue;
        const uint32_t plo = s.defpos[lo.pay], phi = s.defpos[hi.pay];
        if (plo == NONE32 || phi == NONE32) continue;
        const cl_hdr dlo = s.S.hdr[plo], dhi = s.S.hdr[phi];
        if (!(dlo.op == CL_OP_UNPACK64 && has_mod(s, dlo, CL_MB_LO) && dhi.op == CL_OP_UNPACK64 && has_mod(s, dhi, CL_MB_HI))) continue;
        if (!dlo.n_uses || !dhi.n_uses) { fail(s, CL_ST_INDEX_ERROR); continue; }
        opnd slo = get_use(s, dlo, plo, 0), shi = get_use(s, dhi, phi, 0);
        if (!(is_value(slo) && is_value(shi) && slo.pay == shi.pay)) continue;
        if (!h.n_defs) { fail(s, CL_ST_INDEX_ERROR); continue; }
        opnd d = get_def(s, h, i, 0);
        if (!is_value(d)) { fail(s, CL_ST_ATTRIBUTE_ERROR); continue; }
        if (d.pay < s.cap.V) s.redirect[d.pay] = slo.pay;
        mine++;
    }
    const uint32_t changed = g.sum(mine);
    g.sync();
    if (status(s) || !changed) return changed;
    GFOR(g, i, s.n) if (i < s.n) {
        const cl_hdr h = s.S.hdr[i];
        const unsigned u0 = use0(h);
        for (unsigned k = 0; k < h.n_uses; k++) {
            opnd u = get_slot(s, h, i, u0 + k);
            if (is_value(u)) { const uint32_t f = final_of(s, u.pay); if (f != u.pay) { u.pay = f; set_slot(s, h, i, u0 + k, u); } }
            else if (kind_of(u.tag) == CL_K_MEMREF) {
                cl_memref &m = s.mem[u.pay];
                if (kind_of(m.base_tag) == CL_K_VALUE) m.base_pay = final_of(s, m.base_pay);
                if (kind_of(m.ureg_tag) == CL_K_VALUE) m.ureg_pay = final_of(s, m.ureg_pay);
            }
        }
        if (has_guard(h)) { opnd gd = get_slot(s, h, i, 0); if (is_value(gd)) { gd.pay = final_of(s, gd.pay); set_slot(s, h, i, 0, gd); } }
    }
    GFOR(g, b, s.nb) if (b < s.nb)
        for (int k = 0; k < 2; k++)
            if (kind_of(s.blk[b].term_tag[k]) == CL_K_VALUE) s.blk[b].term_pay[k] = final_of(s, s.blk[b].term_pay[k]);
    g.sync();
    if (with_dce) remove_dead_pseudo(g, s);
    return changed;
}

/* apply_aggregations (patterns.py:794-802)                                    */
template <class G> CLF void apply_aggregations(const G &g, FS &s) {
    for (uint32_t round = 0; round < s.max_rounds; round++) {
        uint32_t n = apply_patterns(g, s, 0, 2 + round);
        if (status(s)) return;
        n += simplify_packs(g, s);
        if (status(s)) return;
        if (!n) break;
    }
    remove_dead_pseudo(g, s);
}
/* normalize_xmad (patterns.py:805-810)                                        */
template <class G> CLF void normalize_xmad(const G &g, FS &s) {
    if (s.arch != CL_ARCH_SM52) return;
    apply_patterns(g, s, 1, 0);
    if (status(s)) return;
    remove_dead_pseudo(g, s);
}

/* tag_cuda_objects (patterns.py:895-916)                                      */
template <class G> CLF void tag_cuda_objects(const G &g, FS &s) {
    PROF(g, s, PF_TAG);
    GFOR(g, i, s.n) if (i < s.n) {
        cl_hdr h = s.S.hdr[i];
        unsigned kind = 0, use = 7;
        if (h.op == CL_OP_BAR && has_mod(s, h, CL_MB_SYNC)) {
            kind = 1;
            for (unsigned k = 0; k < h.n_uses && k < 7; k++) if (is_imm(get_use(s, h, i, k))) use = k;
        } else if (h.op == CL_OP_WARPSYNC) {
            for (unsigned k = 0; k < h.n_uses && k < 7; k++) {
                opnd u = get_use(s, h, i, k);
                if (is_imm(u)) { if (s.imm[u.pay].bits == 0xFFFFFFFFull) { kind = 2; use = k; } break; }
            }
        } else if (h.op == CL_OP_SHFL)
            kind = 3;
        if (kind) {
            h.flags &= (uint8_t)~(CL_IF_OBJ_MASK | CL_IF_OBJUSE_MASK);
            h.flags |= (uint8_t)(kind << CL_IF_OBJ_SHIFT | use << CL_IF_OBJUSE_SHIFT);
            s.S.hdr[i].flags = h.flags;
        }
    }
    g.sync();
}

/* ------------------------------------------------------- reciprocal chains */
/* normalize_reciprocal (patterns.py:817-888).  The reference is sequential
 * over chains and rebuilds def-use after each one, so chains see each other's
 * bitcasts.  Here: the group builds use lists once (CSR by value, unordered),
 * then lane 0 walks the chains in stream order on a *mutable* view --
 *   users(v) = entries of CSR(root(v)) whose record currently references v
 *              + the inserted bitcasts chained from xhead[v]
 * where root(v) is the original value a renamed value (.bits / .f) took its
 * sites from -- and the group materialises the inserted records at the end. */
CLN bool rec_references(const FS &s, uint32_t i, uint32_t vid) {
    const cl_hdr h = s.S.hdr[i];
    bool r = false;
    for_value_operands(s, h, i, [&](uint32_t v) { r |= v == vid; });
    return r;
}
CLN uint32_t count_sites(const FS &s, uint32_t i, uint32_t vid) {
    const cl_hdr h = s.S.hdr[i];
    uint32_t r = 0;
    for_value_operands(s, h, i, [&](uint32_t v) { r += v == vid; });
    return r;
}
/* iterate users(v): fn(is_extra, index) returns true to stop; a record that
 * references v through several slots may be visited more than once           */
template <class F> CLD bool for_users(const FS &s, uint32_t v, F fn) {
    const uint32_t r = s.root[v];
    for (uint32_t e = s.redirect[r]; e < s.redirect[r + 1]; e++) {
        const uint32_t p = s.site[e];
        if (rec_references(s, p, v) && fn(false, p)) return true;
    }
    for (uint32_t x = s.xhead[v]; x != NONE32; x = s.xr[x].next)
        if (fn(true, x)) return true;
    return false;
}
/* _reaches_f2i (patterns.py:850-860), depth unrolled at compile time         */
template <int D> struct Reach {
    CLM bool run(const FS &s, bool extra, uint32_t idx) {
        const uint16_t op = extra ? s.xr[idx].r.h.op : s.S.hdr[idx].op;
        if (op == CL_OP_F2I) return true;
        uint32_t defs[8]; unsigned nd = 0;
        if (extra) defs[nd++] = s.xr[idx].r.pay[0];
        else {
            const cl_hdr h = s.S.hdr[idx];
            for_value_defs(s, h, idx, [&](uint32_t v) { if (nd < 8) defs[nd++] = v; });
        }
        for (unsigned k = 0; k < nd; k++) {
            const uint32_t v = defs[k];
            if (v >= s.cap.V) continue;
            if (for_users(s, v, [&](bool ex, uint32_t u) { return Reach<D - 1>::run(s, ex, u); })) return true;
        }
        return false;
    }
};
template <> struct Reach<0> {
    CLM bool run(const FS &s, bool extra, uint32_t idx) {
        return (extra ? s.xr[idx].r.h.op : s.S.hdr[idx].op) == CL_OP_F2I;
    }
};
CLD uint32_t block_of(const FS &s, uint32_t pos) {
    uint32_t lo = 0, hi = s.nb;                 /* last b with bo[b] <= pos and non-empty range */
    while (lo + 1 < hi) { const uint32_t mid = (lo + hi) / 2; if (s.bo[mid] <= pos) lo = mid; else hi = mid; }
    return lo;
}

/* read-only dry run of one chain candidate (the MUFU.RCP at position i): its record, the use list of its result,
 * those users (the adds), the use lists of their results and the records two hops on -- what the sequential
 * rewrite and its _reaches_f2i walk will read.  Returns a digest so that the loads are not optimised away.  */
#if CL_DEV
CLN uint32_t recip_touch(const FS &s, uint32_t i, uint32_t nv) {
    uint32_t acc = 0;
    const cl_hdr h = s.S.hdr[i];
    if (!h.n_defs || (h.flags & CL_IF_EXT)) return 0;
    const opnd rcp = get_def(s, h, i, 0);
    if (!is_value(rcp) || rcp.pay >= nv) return 0;
    acc += s.xhead[rcp.pay] + s.root[rcp.pay];
    uint32_t e0 = s.redirect[rcp.pay], e1 = s.redirect[rcp.pay + 1];
    if (e1 > e0 + 16) e1 = e0 + 16;
    for (uint32_t e = e0; e < e1; e++) {
        const uint32_t p = s.site[e];
        const cl_hdr ah = s.S.hdr[p];
        acc += s.S.tag[(size_t)p * 8] + s.S.pay[(size_t)p * 8];
        if ((ah.op != CL_OP_IADD && ah.op != CL_OP_IADD3) || !ah.n_defs || (ah.flags & CL_IF_EXT)) continue;
        const opnd d = get_def(s, ah, p, 0);
        if (!is_value(d) || d.pay >= nv) continue;
        acc += s.xhead[d.pay] + s.root[d.pay];
        uint32_t f0 = s.redirect[d.pay], f1 = s.redirect[d.pay + 1];
        if (f1 > f0 + 16) f1 = f0 + 16;
        for (uint32_t f = f0; f < f1; f++) {
            const uint32_t p2 = s.site[f];
            const cl_hdr h2 = s.S.hdr[p2];
            acc += s.S.tag[(size_t)p2 * 8] + s.S.pay[(size_t)p2 * 8];
            if (!h2.n_defs || (h2.flags & CL_IF_EXT)) continue;
            const opnd d2 = get_def(s, h2, p2, 0);
            if (!is_value(d2) || d2.pay >= nv) continue;
            acc += s.xhead[d2.pay];
            uint32_t q0 = s.redirect[d2.pay], q1 = s.redirect[d2.pay + 1];
            if (q1 > q0 + 8) q1 = q0 + 8;
            for (uint32_t q = q0; q < q1; q++) {
                const uint32_t p3 = s.site[q];
                acc += s.S.hdr[p3].op + s.S.tag[(size_t)p3 * 8] + s.S.pay[(size_t)p3 * 8];
            }
        }
    }
    return acc;
}
#endif

template <class G> CLF void normalize_reciprocal(const G &g, FS &s) {
    PROF(g, s, PF_RECIP);
    /* cheap exit: no MUFU.RCP at all */
    bool mine = false;
    GFOR(g, i, s.n) if (i < s.n) { const cl_hdr h = s.S.hdr[i]; mine |= h.op == CL_OP_MUFU && has_mod(s, h, CL_MB_RCP); }
    if (!g.any(mine)) return;
    build_usecount(g, s);
    /* CSR offsets in redirect[0 .. next_vid] */
    const uint32_t nv = s.next_vid;
    uint32_t run = 0;
    GFOR(g, v, nv + 1) {
        const uint32_t x = v < nv ? s.usecnt[v] : 0u;
        uint32_t t;
        const uint32_t o = g.exscan(x, t);
        if (v <= nv) s.redirect[v] = run + o;
        run += t;
    }
    if (run > s.cap.U || nv + 1 > s.cap.V) { fail(s, CL_ST_CAPACITY); g.sync(); return; }
    g.sync();
    GFOR(g, v, s.cap.V) if (v < s.cap.V) { s.xhead[v] = NONE32; s.root[v] = v; if (v < nv) s.usecnt[v] = s.redirect[v]; }
    GFOR(g, i, s.n) if (i < s.n) { s.keep[i] = 0; s.inscnt[i] = 0; }       /* before / after counts */
    g.sync();
    GFOR(g, i, s.n) if (i < s.n) {
        const cl_hdr h = s.S.hdr[i];
        for_value_operands(s, h, i, [&](uint32_t v) { if (v < nv) s.site[p_add(s, &s.usecnt[v], 1u)] = i; });
    }
    g.sync();
    uint32_t nx = 0, n_events = 0, vid = s.next_vid, iid = s.next_iid;
    /* the MUFU.RCP records fed by an I2F, in stream order: found by all lanes (ordered compaction into outpos[],
     * free until the materialisation below), so that the sequential part walks a handful of candidates instead
     * of every record of the function (a 20 000-record block spent 2/3 of its stage in that walk).  The test
     * reads nothing a chain rewrite changes: rewrites touch the uses of adds and of their users' operands, and a
     * MUFU whose source is an add result is no candidate before (IADD) or after (BITCAST) the rewrite.        */
    uint32_t n_cand = 0;
    GFOR(g, i, s.n) {
        bool c = false;
        if (i < s.n) {
            const cl_hdr h = s.S.hdr[i];
            if (h.op == CL_OP_MUFU && has_mod(s, h, CL_MB_RCP) && h.n_uses) {
                const opnd src = get_use(s, h, i, 0);
                if (is_value(src) && src.pay < s.cap.V) {
                    /* du.def_inst of the source: original values only (bitcast results never feed a MUFU's I2F test) */
                    const uint32_t dp = src.pay < nv ? s.defpos[src.pay] : NONE32;
                    c = dp != NONE32 && s.S.hdr[dp].op == CL_OP_I2F;
                }
            }
        }
        uint32_t t;
        const uint32_t o = g.flag_exscan(c, t);
        if (c) s.outpos[n_cand + o] = i;
        n_cand += t;
    }
    g.sync();
    /* The chains are rewritten by lane 0 in stream order (each sees the rewrites before it); one chain is ~70
     * dependent loads, i.e. DRAM latency times 70.  The other warps run ahead of it: while lane 0 rewrites one
     * batch of candidates they read what the next batch will read (recip_touch: a dry run without side effects),
     * so that lane 0 finds its records, use lists and users in L1.                                           */
    constexpr uint32_t BATCH = 64;
    const uint32_t h0 = g.size > 32 ? 32u : 1u, nh = g.size > h0 ? (g.size - h0 < BATCH ? g.size - h0 : BATCH) : 0u;
    auto touch = [&](uint32_t cb) {
#if CL_DEV
        if (g.rank >= h0 && g.rank < h0 + nh)
            for (uint32_t k = g.rank - h0; k < BATCH && cb + k < n_cand; k += nh) {
                const uint32_t acc = recip_touch(s, s.outpos[cb + k], nv);
                asm volatile("" ::"r"(acc));
            }
#else
        (void)cb; (void)h0; (void)nh;
#endif
    };
    touch(0);
    g.sync();
    {
    PROF(g, s, PF_SETUP);                       /* profile build: the sequential part of the pass */
    for (uint32_t cb = 0; cb < n_cand; cb += BATCH) {
      if (g.rank != 0) touch(cb + BATCH);
      else {
        const uint32_t ce = cb + BATCH < n_cand ? cb + BATCH : n_cand;
        for (uint32_t ci_ = cb; ci_ < ce && !status(s); ci_++) {
            {
                const uint32_t i = s.outpos[ci_], bi = block_of(s, i);
                const cl_hdr h = s.S.hdr[i];
                if (!h.n_defs) { fail(s, CL_ST_INDEX_ERROR); break; }
                opnd rcp = get_def(s, h, i, 0);
                if (!is_value(rcp)) { fail(s, CL_ST_ATTRIBUTE_ERROR); break; }
                /* adds = user sites of rcp that are IADD/IADD3 with an Imm use, stream order :835-837.
                 * The list is fixed before the first chain of this MUFU is rewritten.          */
                uint32_t *adds = s.cand, *uniq = s.sel_at;          /* scratch: [I] each */
                uint32_t n_adds = 0, n_uniq = 0;
                for_users(s, rcp.pay, [&](bool ex, uint32_t u) {
                    if (ex) return false;
                    const cl_hdr ah = s.S.hdr[u];
                    if (ah.op != CL_OP_IADD && ah.op != CL_OP_IADD3) return false;
                    bool any_imm = false;
                    for (unsigned k = 0; k < ah.n_uses; k++) any_imm |= is_imm(get_use(s, ah, u, k));
                    if (!any_imm) return false;
                    /* the CSR lists are unordered: insertion-sort the (few) distinct adds */
                    uint32_t j = n_uniq;
                    for (uint32_t q = 0; q < n_uniq; q++) if (uniq[q] == u) return false;
                    if (n_uniq >= s.cap.I) return false;
                    while (j > 0 && uniq[j - 1] > u) { uniq[j] = uniq[j - 1]; j--; }
                    uniq[j] = u;
                    n_uniq++;
                    return false;
                });
                for (uint32_t q = 0; q < n_uniq; q++) {              /* one entry per use site */
                    const uint32_t mult = count_sites(s, uniq[q], rcp.pay);
                    for (uint32_t m = 0; m < mult && n_adds < s.cap.I; m++) adds[n_adds++] = uniq[q];
                }
                for (uint32_t ai = 0; ai < n_adds && !status(s); ai++) {
                    const uint32_t a = adds[ai];
                    if (!Reach<3>::run(s, false, a)) continue;
                    if (nx + 2 > s.cap.X || vid + 2 > s.cap.V) { fail(s, CL_ST_CAPACITY); break; }
                    const cl_hdr ah = s.S.hdr[a];
                    /* _insert_reciprocal_bitcasts :863-888 */
                    const uint32_t vi = vid++;
                    s.alive[vi] = 1; s.origin[vi] = CL_ORG_BITS | rcp.pay; s.root[vi] = s.root[rcp.pay]; s.xhead[vi] = NONE32;
                    XRec &ci = s.xr[nx];
                    memset(&ci.r, 0, sizeof ci.r);
                    ci.r.h.iid = iid++; ci.r.h.op = CL_OP_BITCAST; ci.r.h.modset = CL_MS_F2I; ci.r.h.n_defs = 1; ci.r.h.n_uses = 1;
                    ci.r.tag[0] = CL_K_VALUE; ci.r.pay[0] = vi; ci.r.tag[1] = CL_K_VALUE; ci.r.pay[1] = rcp.pay;
                    s.def_iid[vi] = (int32_t)ci.r.h.iid;
                    ci.anchor = a; ci.after = 0; ci.order = s.keep[a]++;
                    ci.next = s.xhead[rcp.pay]; s.xhead[rcp.pay] = nx;
                    nx++;
                    for (unsigned k = 0; k < ah.n_uses; k++) {
                        opnd x = get_use(s, ah, a, k);
                        if (is_value(x) && x.pay == rcp.pay) { x.pay = vi; set_slot(s, ah, a, use0(ah) + k, x); }
                    }
                    if (!ah.n_defs) { fail(s, CL_ST_INDEX_ERROR); break; }
                    opnd add_ref = get_def(s, ah, a, 0);
                    if (!is_value(add_ref)) { fail(s, CL_ST_ATTRIBUTE_ERROR); break; }
                    const uint32_t vf = vid++;
                    s.alive[vf] = 1; s.origin[vf] = CL_ORG_F | add_ref.pay; s.root[vf] = s.root[add_ref.pay]; s.xhead[vf] = NONE32;
                    const uint32_t co_i = nx;
                    XRec &co = s.xr[nx];
                    memset(&co.r, 0, sizeof co.r);
                    co.r.h.iid = iid++; co.r.h.op = CL_OP_BITCAST; co.r.h.modset = CL_MS_I2F; co.r.h.n_defs = 1; co.r.h.n_uses = 1;
                    co.r.tag[0] = CL_K_VALUE; co.r.pay[0] = vf; co.r.tag[1] = CL_K_VALUE; co.r.pay[1] = add_ref.pay;
                    s.def_iid[vf] = (int32_t)co.r.h.iid;
                    co.anchor = a; co.after = 1; co.order = s.inscnt[a]++;
                    nx++;
                    /* every current user of add_def (top-level uses only) now reads vf :878-883 */
                    const uint32_t r0 = s.root[add_ref.pay];
                    for (uint32_t e = s.redirect[r0]; e < s.redirect[r0 + 1]; e++) {
                        const uint32_t p = s.site[e];
                        const cl_hdr uh = s.S.hdr[p];
                        for (unsigned k = 0; k < uh.n_uses; k++) {
                            opnd x = get_use(s, uh, p, k);
                            if (is_value(x) && x.pay == add_ref.pay) { x.pay = vf; set_slot(s, uh, p, use0(uh) + k, x); }
                        }
                    }
                    /* earlier bitcasts reading add_def move over too (the add was rewritten twice) */
                    for (uint32_t x = s.xhead[add_ref.pay]; x != NONE32;) {
                        const uint32_t nxt = s.xr[x].next;
                        s.xr[x].r.pay[1] = vf;
                        s.xr[x].next = s.xhead[vf]; s.xhead[vf] = x;
                        x = nxt;
                    }
                    s.xhead[add_ref.pay] = co_i;
                    s.xr[co_i].next = NONE32;
                    if (block_of(s, a) != bi) { fail(s, CL_ST_KEY_ERROR); break; }            /* pos[add.iid] :886 */
                    push_event(s, 1u << 28, CL_EV_BOUNDARY, n_events++, rcp.pay, ah.iid, 0, 0);
                }
            }
        }
      }
      g.sync();
    }
    }
    nx = g.bcast0(nx); vid = g.bcast0(vid); iid = g.bcast0(iid);
    if (status(s)) return;
    s.next_vid = vid; s.next_iid = iid;
    if (nx == 0) return;
    if (s.n + nx > s.cap.I) { fail(s, CL_ST_CAPACITY); g.sync(); return; }
    /* materialise: right-align, then expand leftwards in order */
    PROF(g, s, 15);
    const uint32_t n = s.n, shift = s.cap.I - n;
    uint32_t run2 = 0;
    GFOR(g, i, n) {
        const uint32_t x = i < n ? 1u + s.keep[i] + s.inscnt[i] : 0u;
        uint32_t t;
        const uint32_t o = g.exscan(x, t);
        if (i < n) s.outpos[i] = run2 + o;
        run2 += t;
    }
    g.sync();
    GFOR(g, b, s.nb + 1) if (b <= s.nb) { const uint32_t old = s.bo[b]; s.bo2[b] = old < n ? s.outpos[old] : run2; }
    move_recs(g, s, shift, 0, n);
    /* outpos is increasing and outpos[i] <= i + inserted-before, so a chunked forward move is safe:
     * destination of record i never passes the source of record i (shift >= nx).            */
    const uint32_t chunks = (n + g.size - 1) / g.size;
    for (uint32_t c = 0; c < chunks; c++) {
        const uint32_t i = c * g.size + g.rank;
        Rec r;
        if (i < n) ld_rec(s, shift + i, r);
        g.sync();
        if (i < n) st_rec(s, s.outpos[i] + s.keep[i], r);
        g.sync();
    }
    GFOR(g, x, nx) if (x < nx) {
        const XRec &e = s.xr[x];
        const uint32_t base = s.outpos[e.anchor];
        const uint32_t at = e.after ? base + s.keep[e.anchor] + 1u + (s.inscnt[e.anchor] - 1u - e.order) : base + e.order;
        st_rec(s, at, e.r);
    }
    { uint32_t *t = s.bo; s.bo = s.bo2; s.bo2 = t; }
    s.n = run2;
    g.sync();
}

/* the four calls of pipeline.py:165-169 on one resident function             */
template <class G> CLF void run_postssa(const G &g, FS &s) {
    if ((s.passes & CL_PASS_XMAD) && !status(s)) normalize_xmad(g, s);
    if ((s.passes & CL_PASS_RECIPROCAL) && !status(s)) normalize_reciprocal(g, s);
    if ((s.passes & CL_PASS_AGGREGATE) && !status(s)) apply_aggregations(g, s);
    if ((s.passes & CL_PASS_TAG) && !status(s)) tag_cuda_objects(g, s);
}
/* match_patterns + select_matches only                                       */
template <class G> CLF void run_match_only(const G &g, FS &s) {
    const unsigned table = (s.passes & CL_PASS_MATCH_XMAD) ? 1 : 0;
    setup_classes(s, table);
    build_usecount(g, s);
    for (uint32_t bi = 0; bi < s.nb; bi++) {
        const uint32_t lo = s.bo[bi], n = s.bo[bi + 1] - lo;
        if (n == 0) continue;
        const uint32_t nm = match_block(g, s, lo, n, table);
        if (status(s)) return;
        if (nm == 0) continue;
        const uint32_t ns = select_block(g, s, n, nm, bi, 0);
        if (status(s)) return;
        if (g.rank == 0) {
            for (uint32_t m = 0; m < nm; m++) s.st_matches[s.mt[m].pat]++;
            for (uint32_t j = 0; j < ns; j++) s.st_selected[s.sel[j].pat]++;
        }
        emit_match_events(g, s, bi, nm, 0, ns);
        g.sync();
    }
}

/* ------------------------------------------------------------- raw stage */
/* The function is one block holding fn.raw_instructions (register operands,
 * guards in slot 0).  Both passes expand the stream in place: count, scan,
 * right-align, move.                                                        */

/* expand the stream: record i moves to outpos[i] + inscnt[i]; the inscnt[i]
 * slots before it are left for the caller to fill                           */
template <class G> CLF uint32_t expand_stream(const G &g, FS &s) {
    const uint32_t n = s.n;
    uint32_t run = 0;
    GFOR(g, i, n) {
        const uint32_t x = i < n ? 1u + s.inscnt[i] : 0u;
        uint32_t t;
        const uint32_t o = g.exscan(x, t);
        if (i < n) s.outpos[i] = run + o;
        run += t;
    }
    if (run > s.cap.I) { fail(s, CL_ST_CAPACITY); g.sync(); return 0; }
    g.sync();
    if (run == n) return n;
    const uint32_t shift = s.cap.I - n;
    move_recs(g, s, shift, 0, n);
    const uint32_t chunks = (n + g.size - 1) / g.size;
    for (uint32_t c = 0; c < chunks; c++) {
        const uint32_t i = c * g.size + g.rank;
        Rec r;
        if (i < n) ld_rec(s, shift + i, r);
        g.sync();
        if (i < n) st_rec(s, s.outpos[i] + s.inscnt[i], r);
        g.sync();
    }
    GFOR(g, b, s.nb + 1) if (b <= s.nb) s.bo[b] = b == 0 ? 0u : run;     /* raw corpora: one block */
    s.n = run;
    g.sync();
    return run;
}

/* normalize_instruction (frontend.py:523-548): PT aux defs dropped; `.X4`
 * loads/stores get an explicit SHL of the address base into a fresh R1000+
 * temporary (temps, iids and immediates numbered in stream order by scan).  */
template <class G> CLF void raw_x4(const G &g, FS &s) {
    const uint32_t n = s.n;
    GFOR(g, i, n) if (i < n) {
        cl_hdr h = s.S.hdr[i];
        if (h.n_aux) {                                        /* :527-528 */
            const unsigned a0 = aux0(h), total = a0 + h.n_aux + h.n_uses;
            unsigned w = a0, na = 0;
            for (unsigned k = a0; k < total; k++) {
                const opnd o = get_slot(s, h, i, k);
                const bool is_aux = k < a0 + h.n_aux;
                if (is_aux && kind_of(o.tag) == CL_K_PRED && o.pay == CL_PT_INDEX) continue;
                if (w != k) set_slot(s, h, i, w, o);
                w++;
                na += is_aux;
            }
            opnd none; none.tag = 0; none.pay = 0;
            if (!(h.flags & CL_IF_EXT)) for (unsigned k = w; k < 8; k++) set_slot(s, h, i, k, none);
            if (na != h.n_aux) { h.n_aux = (uint8_t)na; s.S.hdr[i].n_aux = (uint8_t)na; }
        }
        unsigned want = 0;
        if (has_mod(s, h, CL_MB_X4) && h.op < CL_OP__COUNT && (s.opflags[h.op] & CL_OPF_LDST))
            for (unsigned k = 0; k < h.n_uses; k++) {
                const opnd u = get_use(s, h, i, k);
                if (kind_of(u.tag) != CL_K_MEMREF) continue;
                want = kind_of(s.mem[u.pay].base_tag) == CL_K_REG;      /* first MemRef only :534 */
                break;
            }
        s.inscnt[i] = (uint8_t)want;
    }
    g.sync();
    /* rank of every scaled access = its temp / iid / immediate number */
    uint32_t run = 0;
    GFOR(g, i, n) {
        const uint32_t x = i < n ? s.inscnt[i] : 0u;
        uint32_t t;
        const uint32_t o = g.exscan(x, t);
        if (i < n) s.cand[i] = run + o;
        run += t;
    }
    if (s.n_imm + run > s.cap.Q) { fail(s, CL_ST_CAPACITY); g.sync(); return; }
    g.sync();
    if (run == 0) return;
    if (expand_stream(g, s) == 0 && status(s)) return;
    GFOR(g, i, n) if (i < n && s.inscnt[i]) {
        const uint32_t at = s.outpos[i] + 1u;                 /* the access itself; the SHL goes right before */
        cl_hdr h = s.S.hdr[at];
        const uint32_t k = s.cand[i];
        const uint32_t tmp = s.next_temp + k;
        uint32_t mi = 0;
        for (unsigned u = 0; u < h.n_uses; u++) {
            const opnd o = get_use(s, h, at, u);
            if (kind_of(o.tag) == CL_K_MEMREF) { mi = o.pay; break; }
        }
        cl_memref &m = s.mem[mi];
        cl_imm two; two.bits = 2; two.text = 2;
        s.imm[s.n_imm + k] = two;
        Rec shl;
        shl.h.iid = s.next_iid + k; shl.h.op = CL_OP_SHL; shl.h.modset = CL_MS_NONE;
        shl.h.n_defs = 1; shl.h.n_aux = 0; shl.h.n_uses = 2; shl.h.flags = CL_IF_SYNTH;
        shl.h.ext = (h.flags & CL_IF_SYNTH) && !(h.flags & CL_IF_EXT) ? h.ext : h.iid;   /* shares inst.raw */
        for (unsigned q = 0; q < 8; q++) { shl.tag[q] = 0; shl.pay[q] = 0; }
        unsigned q = 0;
        if (has_guard(h)) { const opnd gd = get_slot(s, h, at, 0); shl.h.flags |= CL_IF_GUARD; shl.tag[0] = gd.tag; shl.pay[0] = gd.pay; q = 1; }
        shl.tag[q] = CL_K_REG; shl.pay[q] = tmp | 1u << 16; q++;
        shl.tag[q] = m.base_tag; shl.pay[q] = m.base_pay; q++;
        shl.tag[q] = (uint16_t)(CL_K_IMM | CL_T_IMM_HEXTEXT); shl.pay[q] = s.n_imm + k;
        st_rec(s, at - 1u, shl);
        m.base_tag = CL_K_REG;                                /* Reg(tmp, old width): flags cleared */
        m.base_pay = tmp | (m.base_pay & 0xFFFF0000u);
        s.S.hdr[at].modset = s.ms[h.modset].minus_x4;
    }
    s.next_temp += run; s.next_iid += run; s.n_imm += run;
    g.sync();
}

/* substitute_special_registers (frontend.py:697-722): constant-bank aliases of
 * special registers become reads of one S2R per (function, offset), inserted
 * before the first instruction that uses it; temporaries are numbered in
 * order of first encounter (instruction, then use index).                   */
static constexpr int MAX_SR = 16;
template <class G> CLF void raw_sr(const G &g, FS &s, const cl_sr_entry *map, uint32_t n_map) {
    uint32_t mine[MAX_SR];
    unsigned nmine = 0;
    for (uint32_t k = 0; k < n_map && nmine < (unsigned)MAX_SR; k++) if (map[k].arch == s.arch) mine[nmine++] = k;
    if (!nmine) return;
    const uint32_t n = s.n;
    uint32_t *first = s.redirect;                            /* [MAX_SR] first encounter: pos << 8 | use */
    GFOR(g, k, nmine) if (k < nmine) first[k] = NONE32;
    GFOR(g, i, n) if (i < n) s.inscnt[i] = 0;
    g.sync();
    const uint32_t off_mask = (1u << CL_CM_OFFSET_BITS) - 1u;
    GFOR(g, i, n) if (i < n) {
        const cl_hdr h = s.S.hdr[i];
        for (unsigned u = 0; u < h.n_uses; u++) {
            const opnd o = get_use(s, h, i, u);
            if (kind_of(o.tag) != CL_K_CONSTMEM || (o.pay >> CL_CM_OFFSET_BITS)) continue;     /* bank 0 only */
            for (unsigned k = 0; k < nmine; k++)
                if (map[mine[k]].offset == (o.pay & off_mask)) { p_min32(s, &first[k], i << 8 | (u < 255 ? u : 255)); break; }
        }
    }
    g.sync();
    /* order of first encounter -> temp / iid numbers (tiny: every lane computes it) */
    uint32_t ord[MAX_SR], nfound = 0;
    for (unsigned k = 0; k < nmine; k++) {
        if (first[k] == NONE32) { ord[k] = NONE32; continue; }
        uint32_t r = 0;
        for (unsigned j = 0; j < nmine; j++) r += first[j] < first[k];
        ord[k] = r;
        nfound++;
    }
    if (!nfound) return;
    if (g.rank == 0) for (unsigned k = 0; k < nmine; k++) if (ord[k] != NONE32) s.inscnt[first[k] >> 8]++;
    g.sync();
    if (expand_stream(g, s) == 0 && status(s)) return;
    /* S2R records: before their instruction, in encounter order */
    GFOR(g, k, nmine) if (k < nmine && ord[k] != NONE32) {
        const uint32_t p = first[k] >> 8;
        uint32_t before = 0;                                  /* earlier encounters at the same instruction */
        for (unsigned j = 0; j < nmine; j++) before += ord[j] != NONE32 && (first[j] >> 8) == p && first[j] < first[k];
        const uint32_t at = s.outpos[p] + before;
        const cl_hdr h = s.S.hdr[s.outpos[p] + s.inscnt[p]];
        Rec r;
        r.h.iid = s.next_iid + ord[k]; r.h.op = CL_OP_S2R; r.h.modset = CL_MS_NONE;
        r.h.n_defs = 1; r.h.n_aux = 0; r.h.n_uses = 1; r.h.flags = CL_IF_SYNTH;
        r.h.ext = (h.flags & CL_IF_SYNTH) && !(h.flags & CL_IF_EXT) ? h.ext : h.iid;
        for (unsigned q = 0; q < 8; q++) { r.tag[q] = 0; r.pay[q] = 0; }
        r.tag[0] = CL_K_REG; r.pay[0] = (s.next_temp + ord[k]) | 1u << 16;
        r.tag[1] = CL_K_SREG; r.pay[1] = map[mine[k]].sreg;
        st_rec(s, at, r);
    }
    g.sync();
    /* every aliasing use becomes the temporary (flags of the ConstMem kept) */
    GFOR(g, i, s.n) if (i < s.n) {
        const cl_hdr h = s.S.hdr[i];
        if (h.op == CL_OP_S2R && (h.flags & CL_IF_SYNTH)) continue;
        for (unsigned u = 0; u < h.n_uses; u++) {
            const opnd o = get_use(s, h, i, u);
            if (kind_of(o.tag) != CL_K_CONSTMEM || (o.pay >> CL_CM_OFFSET_BITS)) continue;
            for (unsigned k = 0; k < nmine; k++)
                if (map[mine[k]].offset == (o.pay & off_mask)) {
                    opnd r;
                    r.tag = (uint16_t)(CL_K_REG | (o.tag & (CL_T_NEG | CL_T_ABS)) | (o.tag & (3u << CL_T_HALF_SHIFT)));
                    r.pay = (s.next_temp + ord[k]) | 1u << 16;
                    set_slot(s, h, i, use0(h) + u, r);
                    break;
                }
        }
    }
    s.next_temp += nfound; s.next_iid += nfound;
    g.sync();
}

template <class G> CLF void run_raw(const G &g, FS &s, uint32_t passes, const cl_sr_entry *map, uint32_t n_map) {
    if (s.nb != 1) { fail(s, CL_ST_UNSUPPORTED); g.sync(); return; }
    if ((passes & CL_RAW_X4) && !status(s)) raw_x4(g, s);
    if ((passes & CL_RAW_SR) && !status(s)) raw_sr(g, s, map, n_map);
}

} /* namespace clk */

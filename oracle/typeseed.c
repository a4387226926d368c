/* TEST INFRASTRUCTURE -- sequential CPU restatement of the reference's type
 * seeding (typerec.py:78-235 signature_for, :288-345 seed_types), the checker
 * for cl_seed_types of the CUDA library.  Included at the end of oracle.c
 * (one translation unit: it reads the context's copy of the uploaded corpus).
 * Parity is pinned by tests/golden/types.pkl.gz (TypeState of the reference
 * itself, tools/make_types_golden.py).  Never loaded by the product.
 *
 * It follows the reference literally: build the Signature (role, defs[], aux,
 * uses[]) of an instruction as lists, then walk defs / aux defs / uses / guard
 * and the block terminator and narrow.                                      */
#include "../include/culifter_types.h"

#define TS_LINK 0x100u          /* LINK = "link" (typerec.py:30) */
#define TS_NONE 0u              /* None                           */
typedef struct ts_sig { int role; unsigned nd, nu; uint16_t defs[256], uses[260]; uint16_t aux; } ts_sig;

static void ts_fill(uint16_t *a, unsigned *n, uint16_t v, int count) { for (int i = 0; i < count; i++) a[(*n)++] = v; }
static uint16_t ts_load_mask(unsigned width) {                       /* _load_mask :73 */
    return width == 1 ? CL_TY_NUM32 : width == 2 ? CL_TY_NUM64 : width == 4 ? CL_TY_NUM128 : CL_TY_NUM32;
}

typedef struct ts_inst {         /* one record of the uploaded corpus, slots resolved */
    cl_hdr h; const uint16_t *tag; const uint32_t *pay; unsigned g;  /* g: 1 when slot 0 is the guard */
} ts_inst;
static unsigned ts_kind(const ts_inst *r, unsigned slot) { return CL_T_KIND(r->tag[slot]); }

/* signature_for, typerec.py:78-235 */
static void ts_signature(const ts_inst *r, cl_optype ot, cl_modtype mt, uint32_t hint, ts_sig *s) {
    const int nd = r->h.n_defs, nu = r->h.n_uses;
    const unsigned d0 = r->g, u0 = r->g + r->h.n_defs + r->h.n_aux;
    s->role = CL_ROLE_SEED; s->nd = s->nu = 0; s->aux = CL_TY_BOOL;
#define DEFS(v, n) ts_fill(s->defs, &s->nd, (v), (n))
#define USES(v, n) ts_fill(s->uses, &s->nu, (v), (n))
#define CUT(n) do { if ((int)s->nu > (n)) s->nu = (n) < 0 ? 0 : (unsigned)(n); } while (0)
    switch (ot.kind) {
    case CL_SK_FSEL: DEFS(CL_TY_FLOAT32, 1); USES(CL_TY_FLOAT32, 2); USES(CL_TY_BOOL, 1); break;           /* :89 */
    case CL_SK_FALU: DEFS(CL_TY_FLOAT32, nd); USES(CL_TY_FLOAT32, nu); break;                               /* :91 */
    case CL_SK_FCMP: DEFS(CL_TY_BOOL, 1); USES(CL_TY_FLOAT32, 2); USES(CL_TY_BOOL, nu - 2); break;          /* :93 */
    case CL_SK_DALU: DEFS(CL_TY_FLOAT64, nd); USES(CL_TY_FLOAT64, nu); break;
    case CL_SK_DCMP: DEFS(CL_TY_BOOL, 1); USES(CL_TY_FLOAT64, 2); USES(CL_TY_BOOL, nu - 2); break;
    case CL_SK_HALU: DEFS(mt.f16_elem, nd); USES(mt.f16_elem, nu); break;                                   /* :99 */
    case CL_SK_HCMP: DEFS(CL_TY_BOOL, 1); USES(mt.f16_elem, 2); USES(CL_TY_BOOL, nu - 2); break;
    case CL_SK_IMAD:
        if (mt.flags & CL_MT_WIDE) {                                                                          /* :104-107 */
            DEFS(CL_TY_INT64, 1); USES(CL_TY_INT32, 2); USES(CL_TY_INT64, 1); CUT(nu); USES(TS_NONE, nu - 3);
        } else { DEFS(CL_TY_INT32, nd); USES(CL_TY_INT32, nu); }                                              /* :127 */
        break;
    case CL_SK_LOP: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, nd); USES(TS_LINK, nu); break;              /* :109 */
    case CL_SK_SHF: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, nd);                                        /* :112 */
        USES(TS_LINK, 1); USES(CL_TY_INT32, 1); USES(TS_LINK, 1); CUT(nu); USES(TS_NONE, nu - 3); break;
    case CL_SK_SHLR: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, nd); USES(TS_LINK, 1); USES(CL_TY_INT32, 1); CUT(nu); break;
    case CL_SK_IADD3: case CL_SK_IADD: {                                                                      /* :117-120 */
        const int nsrc = ot.kind == CL_SK_IADD ? 2 : 3;
        DEFS(CL_TY_INT32, nd); USES(CL_TY_INT32, nsrc < nu ? nsrc : nu); USES(CL_TY_BOOL, nu - nsrc); break; }
    case CL_SK_LEA: {                                                                                         /* :121-124 */
        const int nsrc = (mt.flags & CL_MT_HI) ? 4 : 3;
        DEFS(CL_TY_INT32, nd); USES(CL_TY_INT32, nsrc < nu ? nsrc : nu); USES(CL_TY_BOOL, nu - nsrc); break; }
    case CL_SK_IALU: DEFS(CL_TY_INT32, nd); USES(CL_TY_INT32, nu); break;
    case CL_SK_ICMP: DEFS(CL_TY_BOOL, 1); USES(CL_TY_INT32, 2); USES(CL_TY_BOOL, nu - 2); break;
    case CL_SK_PRED: DEFS(CL_TY_BOOL, 1); USES(CL_TY_BOOL, nu); break;
    case CL_SK_MOV: {                                                                                         /* :135-139 */
        int any_value = 0; unsigned width = 1; int seen = 0;
        for (int k = 0; k < nu; k++) {
            if (ts_kind(r, u0 + k) == CL_K_VALUE) any_value = 1;
            if (ts_kind(r, u0 + k) == CL_K_CONSTMEM && !seen) { width = CL_T_WIDTH(r->tag[u0 + k]); seen = 1; }
        }
        if (any_value) { s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, nd); USES(TS_LINK, nu); }
        else { DEFS(ts_load_mask(width), nd); USES(TS_NONE, nu); }
        break; }
    case CL_SK_SEL: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, 1); USES(TS_LINK, 2); USES(CL_TY_BOOL, 1); break;
    case CL_SK_SELECT: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, 1); USES(CL_TY_BOOL, 1); USES(TS_LINK, 2); break;
    case CL_SK_PHI: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, 1); USES(TS_LINK, nu); break;
    case CL_SK_SREG: DEFS(CL_TY_INT32, nd); USES(TS_NONE, nu); break;
    case CL_SK_SHUFFLE: s->role = CL_ROLE_TRANSPARENT; DEFS(TS_LINK, 1); USES(TS_LINK, 1); USES(CL_TY_INT32, nu - 1); break;
    case CL_SK_VOTE: DEFS(CL_TY_INT32, nd); USES(CL_TY_BOOL, nu); break;
    case CL_SK_I2F: s->role = CL_ROLE_CONVERSION; DEFS(mt.conv_float, 1); USES(mt.conv_int, nu); break;      /* :154 */
    case CL_SK_F2I: s->role = CL_ROLE_CONVERSION; DEFS(mt.conv_int, 1); USES(mt.conv_float, nu); break;
    case CL_SK_F2F: s->role = CL_ROLE_CONVERSION; DEFS(mt.f2f_dst, 1); USES(mt.f2f_src, nu); break;
    case CL_SK_I2I: s->role = CL_ROLE_CONVERSION; DEFS(CL_TY_INT32, 1); USES(CL_TY_INT32, nu); break;
    case CL_SK_FRND: s->role = CL_ROLE_CONVERSION; DEFS(mt.conv_float, 1); USES(mt.conv_float, nu); break;
    case CL_SK_CAST64: s->role = CL_ROLE_CONVERSION; DEFS(CL_TY_INT64, 1); USES(CL_TY_INT32, 1); break;
    case CL_SK_BITCAST: s->role = CL_ROLE_CONVERSION;                                                         /* :169-174 */
        if (mt.flags & CL_MT_F2I) { DEFS(CL_TY_INT32, 1); USES(CL_TY_FLOAT32, 1); }
        else if (mt.flags & CL_MT_I2F) { DEFS(CL_TY_FLOAT32, 1); USES(CL_TY_INT32, 1); }
        else { DEFS(TS_NONE, nd); USES(TS_NONE, nu); }
        break;
    case CL_SK_LOAD: {                                                                                        /* :176-189 */
        unsigned width = 1;
        for (int k = 0; k < nd; k++) {
            const unsigned kd = ts_kind(r, d0 + k);
            const unsigned w = (kd == CL_K_REG || kd == CL_K_UREG) ? r->pay[d0 + k] >> 16 : 1;
            if (w > width) width = w;
        }
        if (CL_TH_DEFW(hint)) width = CL_TH_DEFW(hint);
        DEFS(ts_load_mask(width), nd);
        for (int k = 0; k < nu; k++)
            USES(ts_kind(r, u0 + k) == CL_K_MEMREF ? ((ot.flags & CL_OT_ADDR64) ? CL_TY_INT64 : CL_TY_INT32) : TS_NONE, 1);
        break; }
    case CL_SK_STORE: {                                                                                       /* :190-198 */
        const unsigned width = CL_TH_DATAW(hint) ? CL_TH_DATAW(hint) : 1;
        const uint16_t elem = (ot.flags & CL_OT_RED) ? mt.atom_elem : ts_load_mask(width);
        for (int k = 0; k < nu; k++)
            USES(ts_kind(r, u0 + k) == CL_K_MEMREF ? ((ot.flags & CL_OT_ADDR64) ? CL_TY_INT64 : CL_TY_INT32) : elem, 1);
        break; }
    case CL_SK_ATOMIC:                                                                                        /* :199-207 */
        DEFS(mt.atom_elem, nd);
        for (int k = 0; k < nu; k++)
            USES(ts_kind(r, u0 + k) == CL_K_MEMREF ? ((ot.flags & CL_OT_ADDR64) ? CL_TY_INT64 : CL_TY_INT32) : mt.atom_elem, 1);
        break;
    case CL_SK_TENSOR: {                                                                                      /* :209-216 */
        const uint16_t acc = (mt.flags & CL_MT_F32) ? CL_TY_FLOAT32 : CL_TY_INT32;
        USES(mt.mma_elem, (int)(CL_TH_NA(hint) + CL_TH_NB(hint))); USES(acc, (int)CL_TH_NC(hint));
        if ((int)s->nu < nu) USES(TS_NONE, nu - (int)s->nu);
        CUT(nu);
        DEFS(acc, nd); break; }
    case CL_SK_IADD364: DEFS(CL_TY_INT64, 1); USES(CL_TY_INT64, nu); break;
    case CL_SK_ISETP64: DEFS(CL_TY_BOOL, 1); USES(CL_TY_INT64, 2); USES(CL_TY_BOOL, nu - 2); break;
    case CL_SK_LEA64: DEFS(CL_TY_INT64, 1); USES(CL_TY_INT64, 2); USES(CL_TY_INT32, 1); CUT(nu); break;
    case CL_SK_IMAD64: DEFS(CL_TY_INT64, 1); USES(CL_TY_INT32, 2); USES(CL_TY_INT64, 1); CUT(nu); break;
    case CL_SK_MOV64: DEFS(CL_TY_NUM64, 1); USES(TS_NONE, nu); break;
    case CL_SK_SH64: DEFS(CL_TY_INT64, 1); USES(CL_TY_INT64, 1); USES(CL_TY_INT32, 1); CUT(nu); break;
    case CL_SK_PACK64: DEFS(CL_TY_NUM64, 1); USES(CL_TY_NUM32, nu); break;
    case CL_SK_PACK128: DEFS(CL_TY_NUM128, 1); USES(CL_TY_NUM32, nu); break;
    case CL_SK_UNPACK64: DEFS(CL_TY_NUM32, 1); USES(CL_TY_NUM64 | CL_TY_NUM128, 1); break;
    case CL_SK_UNPACK128: DEFS(CL_TY_NUM32, 1); USES(CL_TY_NUM128, 1); break;
    default: DEFS(TS_NONE, nd); USES(TS_NONE, nu); break;                                                     /* :234 */
    }
#undef DEFS
#undef USES
#undef CUT
}

typedef struct ts_fn { uint32_t *masks; const uint8_t *alive; uint32_t n_val; int key_error; } ts_fn;
static void ts_narrow(ts_fn *f, uint32_t vid, unsigned mask, int is_def) {           /* narrow, typerec.py:300-305 */
    if (vid >= f->n_val || !f->alive[vid]) { f->key_error = 1; return; }
    const uint32_t drop = (~mask) & 0xFFu;
    f->masks[vid] &= ~(drop | (is_def ? drop << 8 : drop << 16));
}

/* the hint of instruction `iid` of function f: binary search in the function's sorted run, 0 when absent */
static uint32_t ts_hint(const cl_typehints *h, uint32_t f, uint32_t iid) {
    if (!h) return 0;
    uint32_t lo = h->off[f], hi = h->off[f + 1];
    while (lo < hi) { uint32_t mid = lo + (hi - lo) / 2; if (h->iid[mid] < iid) lo = mid + 1; else hi = mid; }
    return lo < h->off[f + 1] && h->iid[lo] == iid ? h->val[lo] : 0;
}

static int ts_seed(const cl_corpus *in, const cl_optype *ops, uint32_t n_ops, const cl_modtype *mods, uint32_t n_mods,
                   const cl_typehints *hints, cl_typeseed *out) {
    ts_sig *sig = malloc(sizeof *sig);
    for (uint32_t f = 0; f < in->n_funcs; f++) {
        ts_fn fs = { out->val_masks + in->val_off[f], in->val_alive + in->val_off[f], in->val_off[f + 1] - in->val_off[f], 0 };
        for (uint32_t v = 0; v < fs.n_val; v++) fs.masks[v] = 0xFFFFFFu;          /* :292-295: TOP */
        for (uint32_t b = in->func_blk_off[f]; b < in->func_blk_off[f + 1]; b++) {  /* block_order(), :307 */
            for (uint32_t i = in->blk_off[b]; i < in->blk_off[b + 1]; i++) {
                ts_inst r; r.h = in->hdr[i]; r.g = (r.h.flags & CL_IF_GUARD) ? 1 : 0;
                if (r.h.flags & CL_IF_EXT) { r.tag = in->ext_tag + in->ext_off[f] + r.h.ext; r.pay = in->ext_pay + in->ext_off[f] + r.h.ext; }
                else { r.tag = in->tag + 8ull * i; r.pay = in->pay + 8ull * i; }
                if (r.h.op >= n_ops || r.h.modset >= n_mods) { free(sig); FAIL("cl_seed_types: opcode / modset id outside the tables"); }
                ts_signature(&r, ops[r.h.op], mods[r.h.modset], ts_hint(hints, f, r.h.iid), sig);
                out->role[i] = (uint8_t)sig->role;                                  /* :311 */
                uint32_t link_def = CL_NO_VALUE; uint16_t link_mask = 0;
                const unsigned d0 = r.g, a0 = d0 + r.h.n_defs, u0 = a0 + r.h.n_aux;
                for (unsigned k = 0; k < r.h.n_defs && k < sig->nd; k++) {          /* :316-322 (zip: shorter list) */
                    if (ts_kind(&r, d0 + k) != CL_K_VALUE) continue;
                    if (sig->defs[k] == TS_LINK) link_def = r.pay[d0 + k];
                    else if (sig->defs[k]) ts_narrow(&fs, r.pay[d0 + k], sig->defs[k], 1);
                }
                for (unsigned k = 0; k < r.h.n_aux; k++)                            /* :323-325 */
                    if (ts_kind(&r, a0 + k) == CL_K_VALUE && sig->aux) ts_narrow(&fs, r.pay[a0 + k], sig->aux, 1);
                for (unsigned k = 0; k < r.h.n_uses; k++) {                         /* :326-333, _slot_values :273 */
                    const unsigned cst = k < sig->nu ? sig->uses[k] : TS_NONE;
                    const unsigned kd = ts_kind(&r, u0 + k);
                    uint32_t ref = CL_NO_VALUE;
                    if (kd == CL_K_VALUE) ref = r.pay[u0 + k];
                    else if (kd == CL_K_MEMREF) {
                        const cl_memref *m = in->mem + in->mem_off[f] + r.pay[u0 + k];
                        if (CL_T_KIND(m->base_tag) == CL_K_VALUE) ref = m->base_pay;
                        if (CL_T_KIND(m->ureg_tag) == CL_K_VALUE) ts_narrow(&fs, m->ureg_pay, CL_TY_INT32, 0);
                    }
                    if (ref == CL_NO_VALUE) continue;
                    if (cst == TS_LINK) link_mask |= (uint16_t)(1u << (k < 15 ? k : 15));
                    else if (cst) ts_narrow(&fs, ref, cst, 0);
                }
                if (r.g && ts_kind(&r, 0) == CL_K_VALUE) ts_narrow(&fs, r.pay[0], CL_TY_BOOL, 0);   /* :334 */
                out->link_def[i] = link_def; out->link_mask[i] = link_mask;
            }
            for (int t = 0; t < 2; t++)                                             /* :342-343 */
                if (CL_T_KIND(in->blk[b].term_tag[t]) == CL_K_VALUE) ts_narrow(&fs, in->blk[b].term_pay[t], CL_TY_BOOL, 0);
        }
        out->status[f] = fs.key_error ? CL_ST_KEY_ERROR : CL_ST_OK;
    }
    free(sig);
    return 0;
}

int cl_seed_types(cl_ctx *c, uint32_t source, const cl_optype *ops, uint32_t n_ops, const cl_modtype *mods, uint32_t n_mods,
                  const cl_typehints *hints, cl_typeseed *out) {
    if (!c->have_in) FAIL("cl_seed_types: no corpus uploaded");
    if (source == CL_SEED_INPUT) {
        struct timespec t0, t1; clock_gettime(CLOCK_MONOTONIC, &t0);
        if (ts_seed(&c->in, ops, n_ops, mods, n_mods, hints, out)) return -1;
        clock_gettime(CLOCK_MONOTONIC, &t1);
        c->last_ms = (float)((t1.tv_sec - t0.tv_sec) * 1e3 + (t1.tv_nsec - t0.tv_nsec) * 1e-6);
        return 0;
    }
    if (source != CL_SEED_RESULT) FAIL("cl_seed_types: unknown source %u", source);
    /* the result of the last run as a dense corpus (what cl_download hands out), then the same walk */
    uint64_t sz[6];
    if (cl_out_sizes(c, sz)) return -1;
    const uint32_t F = c->in.n_funcs, B = c->in.n_blocks;
    cl_corpus r; memset(&r, 0, sizeof r);
    r.func = malloc(sizeof(cl_func) * (F + 1)); r.func_blk_off = malloc(4ull * (F + 1)); r.ext_off = malloc(4ull * (F + 1));
    r.mem_off = malloc(4ull * (F + 1)); r.imm_off = malloc(4ull * (F + 1)); r.val_off = malloc(4ull * (F + 1));
    r.blk = malloc(sizeof(cl_blk) * (B + 1)); r.blk_off = malloc(4ull * (B + 1));
    r.hdr = malloc(sizeof(cl_hdr) * (sz[0] + 1)); r.tag = malloc(16ull * (sz[0] + 1)); r.pay = malloc(32ull * (sz[0] + 1));
    r.ext_tag = malloc(2ull * (sz[1] + 1)); r.ext_pay = malloc(4ull * (sz[1] + 1)); r.mem = malloc(sizeof(cl_memref) * (sz[2] + 1));
    r.imm = malloc(sizeof(cl_imm) * (sz[3] + 1)); r.val_alive = malloc(sz[4] + 1); r.val_def_iid = malloc(4ull * (sz[4] + 1));
    r.val_origin = malloc(4ull * (sz[4] + 1));
    int rc = cl_download(c, &r, NULL);
    if (!rc) {
        struct timespec t0, t1; clock_gettime(CLOCK_MONOTONIC, &t0);
        rc = ts_seed(&r, ops, n_ops, mods, n_mods, hints, out);
        clock_gettime(CLOCK_MONOTONIC, &t1);
        c->last_ms = (float)((t1.tv_sec - t0.tv_sec) * 1e3 + (t1.tv_nsec - t0.tv_nsec) * 1e-6);
    }
    free(r.func); free(r.func_blk_off); free(r.ext_off); free(r.mem_off); free(r.imm_off); free(r.val_off); free(r.blk); free(r.blk_off);
    free(r.hdr); free(r.tag); free(r.pay); free(r.ext_tag); free(r.ext_pay); free(r.mem); free(r.imm); free(r.val_alive);
    free(r.val_def_iid); free(r.val_origin);
    return rc;
}

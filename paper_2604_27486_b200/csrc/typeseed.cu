/* typeseed.cu -- cl_seed_types of include/culifter_types.h on sm_100a:
 * typerec.seed_types (reference typerec.py:288-345) with signature_for
 * (typerec.py:78-235) evaluated per record on the device.
 *
 * One thread per instruction record (grid-stride, 148 SMs x 8 CTAs of 256):
 * the three planes of a record are read once with 128-bit loads (64 B), the
 * constraint of every def / aux def / use slot is computed on the fly from the
 * opcode's signature kind and the modifier-tuple entry (two small tables that
 * stay in L1), and every constrained value is narrowed with ONE 32-bit
 * red.and on its packed mask word (seed | def << 8 | use << 16).  Per record
 * the kernel writes 7 bytes (role, link mask, link def).  A second grid-stride
 * loop narrows the terminator conditions of the blocks.  HBM bound: 64 B read +
 * 7 B written per record + 8 B per value (fill, final read by the copy).
 *
 * Compiled with -DCL_SIM by g++ (tests/sim) the kernels become loops: logic
 * checks without a GPU.  Never a fallback of the product.                    */
#include "../../include/culifter_types.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>

#if defined(__CUDACC__) && !defined(CL_SIM)
#include <cuda_runtime.h>
#define TS_CUDA 1
#define TS_HD __host__ __device__ __forceinline__
#define TS_D __device__ __forceinline__
#define TS_M __host__ __device__ __forceinline__
#else
#define TS_CUDA 0
#define TS_HD static inline
#define TS_D static inline
#define TS_M inline
struct uint4 { uint32_t x, y, z, w; };
#endif

/* culifter.cu: device view of the corpus a context holds (not part of the C ABI) */
extern "C" int cli_corpus_view(cl_ctx *c, uint32_t source, cl_corpus *view, uint64_t counts[2], void **stream, float **last_ms);
extern "C" void cli_set_error(const char *msg);
#define FAIL(...) do { char b_[400]; snprintf(b_, sizeof b_, __VA_ARGS__); cli_set_error(b_); return -1; } while (0)

#define TS_LINK 0x100u

struct TsArgs {
    cl_corpus in;                    /* device pointers */
    const uint32_t *func_rec_off;    /* [F+1] first record of every function */
    const cl_optype *ops; const cl_modtype *mods;
    const uint32_t *hint_off, *hint_iid, *hint_val;   /* cl_typehints on the device, hint_off == nullptr: none */
    uint32_t n_ops, n_mods, n_inst, n_val;
    uint32_t *val_masks; uint8_t *role; uint16_t *link_mask; uint32_t *link_def; uint8_t *status;
    uint32_t *bad;                   /* set when a record names an id outside the tables */
};

/* the hint of instruction `iid` of function f (binary search in the function's sorted run), 0 when absent */
TS_HD uint32_t ts_hint(const TsArgs &a, uint32_t f, uint32_t iid) {
    if (!a.hint_off) return 0;
    uint32_t lo = a.hint_off[f];
    const uint32_t end = a.hint_off[f + 1];
    uint32_t hi = end;
    while (lo < hi) { const uint32_t mid = lo + ((hi - lo) >> 1); if (a.hint_iid[mid] < iid) lo = mid + 1; else hi = mid; }
    return lo < end && a.hint_iid[lo] == iid ? a.hint_val[lo] : 0u;
}

TS_HD uint32_t ts_load_mask(uint32_t w) { return w == 2 ? CL_TY_NUM64 : w == 4 ? CL_TY_NUM128 : CL_TY_NUM32; }

/* the slots of one record, wherever they live */
struct TsRec {
    cl_hdr h; uint32_t g, f;
    uint16_t tag8[8]; uint32_t pay8[8];
    const uint16_t *xt; const uint32_t *xp;      /* ext region when CL_IF_EXT */
};

/* Signature.defs[k] (typerec.py:87-234): 0 = None, TS_LINK, else a mask.  Entries past the signature's list are
 * None (zip stops at the shorter list, typerec.py:316).                                                         */
TS_HD uint32_t ts_def_c(uint32_t kind, uint32_t k, cl_modtype mt, uint32_t loadw, uint32_t accw) {
    const bool first = k == 0;
    switch (kind) {
    case CL_SK_FALU: return CL_TY_FLOAT32;
    case CL_SK_FSEL: return first ? CL_TY_FLOAT32 : 0;
    case CL_SK_FCMP: case CL_SK_DCMP: case CL_SK_HCMP: case CL_SK_ICMP: case CL_SK_PRED: case CL_SK_ISETP64: return first ? CL_TY_BOOL : 0;
    case CL_SK_DALU: return CL_TY_FLOAT64;
    case CL_SK_HALU: return mt.f16_elem;
    case CL_SK_IMAD: return (mt.flags & CL_MT_WIDE) ? (first ? CL_TY_INT64 : 0) : CL_TY_INT32;
    case CL_SK_LOP: case CL_SK_SHF: case CL_SK_SHLR: return TS_LINK;
    case CL_SK_IADD3: case CL_SK_IADD: case CL_SK_LEA: case CL_SK_IALU: case CL_SK_SREG: case CL_SK_VOTE: return CL_TY_INT32;
    case CL_SK_MOV: return loadw;                       /* TS_LINK when a use is a value, else _load_mask(ConstMem width) */
    case CL_SK_SEL: case CL_SK_SELECT: case CL_SK_PHI: case CL_SK_SHUFFLE: return first ? TS_LINK : 0;
    case CL_SK_I2F: case CL_SK_FRND: return first ? mt.conv_float : 0;
    case CL_SK_F2I: return first ? mt.conv_int : 0;
    case CL_SK_F2F: return first ? mt.f2f_dst : 0;
    case CL_SK_I2I: return first ? CL_TY_INT32 : 0;
    case CL_SK_CAST64: case CL_SK_IADD364: case CL_SK_LEA64: case CL_SK_IMAD64: case CL_SK_SH64: return first ? CL_TY_INT64 : 0;
    case CL_SK_BITCAST: return !first ? 0 : (mt.flags & CL_MT_F2I) ? CL_TY_INT32 : (mt.flags & CL_MT_I2F) ? CL_TY_FLOAT32 : 0;
    case CL_SK_LOAD: return loadw;
    case CL_SK_ATOMIC: return mt.atom_elem;
    case CL_SK_TENSOR: return accw;
    case CL_SK_MOV64: case CL_SK_PACK64: return first ? CL_TY_NUM64 : 0;
    case CL_SK_PACK128: return first ? CL_TY_NUM128 : 0;
    case CL_SK_UNPACK64: case CL_SK_UNPACK128: return first ? CL_TY_NUM32 : 0;
    default: return 0;
    }
}

/* Signature.uses[k] for a use that is not decided by its operand kind (MemRef uses of the memory opcodes are) */
TS_HD uint32_t ts_use_c(uint32_t kind, uint32_t k, uint32_t nu, cl_optype ot, cl_modtype mt, uint32_t movlink,
                        uint32_t elem, uint32_t accw, uint32_t hint) {
    switch (kind) {
    case CL_SK_FALU: return CL_TY_FLOAT32;
    case CL_SK_FSEL: return k < 2 ? CL_TY_FLOAT32 : k == 2 ? CL_TY_BOOL : 0;
    case CL_SK_FCMP: return k < 2 ? CL_TY_FLOAT32 : CL_TY_BOOL;
    case CL_SK_DALU: return CL_TY_FLOAT64;
    case CL_SK_DCMP: return k < 2 ? CL_TY_FLOAT64 : CL_TY_BOOL;
    case CL_SK_HALU: return mt.f16_elem;
    case CL_SK_HCMP: return k < 2 ? mt.f16_elem : CL_TY_BOOL;
    case CL_SK_IMAD: return !(mt.flags & CL_MT_WIDE) ? CL_TY_INT32 : k < 2 ? CL_TY_INT32 : k == 2 ? CL_TY_INT64 : 0;
    case CL_SK_LOP: case CL_SK_PHI: return TS_LINK;
    case CL_SK_SHF: return k == 0 || k == 2 ? TS_LINK : k == 1 ? CL_TY_INT32 : 0;
    case CL_SK_SHLR: return k == 0 ? TS_LINK : k == 1 ? CL_TY_INT32 : 0;
    case CL_SK_IADD3: return k < 3 ? CL_TY_INT32 : CL_TY_BOOL;
    case CL_SK_IADD: return k < 2 ? CL_TY_INT32 : CL_TY_BOOL;
    case CL_SK_LEA: return k < ((mt.flags & CL_MT_HI) ? 4u : 3u) ? CL_TY_INT32 : CL_TY_BOOL;
    case CL_SK_IALU: return CL_TY_INT32;
    case CL_SK_ICMP: return k < 2 ? CL_TY_INT32 : CL_TY_BOOL;
    case CL_SK_PRED: case CL_SK_VOTE: return CL_TY_BOOL;
    case CL_SK_MOV: return movlink;
    case CL_SK_SEL: return k < 2 ? TS_LINK : k == 2 ? CL_TY_BOOL : 0;
    case CL_SK_SELECT: return k == 0 ? CL_TY_BOOL : k < 3 ? TS_LINK : 0;
    case CL_SK_SHUFFLE: return k == 0 ? TS_LINK : CL_TY_INT32;
    case CL_SK_I2F: return mt.conv_int;
    case CL_SK_F2I: case CL_SK_FRND: return mt.conv_float;
    case CL_SK_F2F: return mt.f2f_src;
    case CL_SK_I2I: return CL_TY_INT32;
    case CL_SK_CAST64: return k == 0 ? CL_TY_INT32 : 0;
    case CL_SK_BITCAST: return k != 0 ? 0 : (mt.flags & CL_MT_F2I) ? CL_TY_FLOAT32 : (mt.flags & CL_MT_I2F) ? CL_TY_INT32 : 0;
    case CL_SK_STORE: case CL_SK_ATOMIC: return elem;
    case CL_SK_TENSOR: { const uint32_t ab = CL_TH_NA(hint) + CL_TH_NB(hint); return k < ab ? mt.mma_elem : k < ab + CL_TH_NC(hint) ? accw : 0; }
    case CL_SK_IADD364: return CL_TY_INT64;
    case CL_SK_ISETP64: return k < 2 ? CL_TY_INT64 : CL_TY_BOOL;
    case CL_SK_LEA64: return k < 2 ? CL_TY_INT64 : k == 2 ? CL_TY_INT32 : 0;
    case CL_SK_IMAD64: return k < 2 ? CL_TY_INT32 : k == 2 ? CL_TY_INT64 : 0;
    case CL_SK_SH64: return k == 0 ? CL_TY_INT64 : k == 1 ? CL_TY_INT32 : 0;
    case CL_SK_PACK64: case CL_SK_PACK128: return CL_TY_NUM32;
    case CL_SK_UNPACK64: return k == 0 ? (CL_TY_NUM64 | CL_TY_NUM128) : 0;
    case CL_SK_UNPACK128: return k == 0 ? CL_TY_NUM128 : 0;
    default: (void)nu; (void)ot; return 0;          /* NONE, SREG, MOV64, LOAD (non-MemRef uses) */
    }
}

TS_D void ts_and(uint32_t *p, uint32_t v) {
#if TS_CUDA
    atomicAnd(p, v);          /* result unused: compiles to RED.AND */
#else
    *p &= v;
#endif
}
/* narrow (typerec.py:300-305) */
TS_D void ts_narrow(const TsArgs &a, uint32_t f, uint32_t v0, uint32_t nv, uint32_t vid, uint32_t mask, bool is_def) {
    if (vid >= nv || !a.in.val_alive[v0 + vid]) { a.status[f] = CL_ST_KEY_ERROR; return; }
    const uint32_t drop = ~mask & 0xFFu;
    if (drop) ts_and(a.val_masks + v0 + vid, ~(drop | (is_def ? drop << 8 : drop << 16)));
}

/* One record.  EXT = false: the 8 inline slots sit in registers and every slot loop is unrolled over the absolute
 * slot index (no local-memory array); EXT = true (more than 8 slots: wide PHIs, tensor ops): slots are read from
 * the function's overflow region.                                                                              */
template <bool EXT> TS_D void ts_slots(const TsArgs &a, uint32_t i, uint32_t f, const TsRec &r) {
    const cl_optype ot = a.ops[r.h.op];
    const cl_modtype mt = a.mods[r.h.modset];
    /* only loads, stores and tensor ops read Instruction.meta */
    const uint32_t hint = (ot.kind == CL_SK_LOAD || ot.kind == CL_SK_STORE || ot.kind == CL_SK_TENSOR) ? ts_hint(a, f, r.h.iid) : 0u;
    const uint32_t nd = r.h.n_defs, na = r.h.n_aux, nu = r.h.n_uses;
    const uint32_t d0 = r.g, a0 = d0 + nd, u0 = a0 + na, total = u0 + nu;
    const uint32_t v0 = a.in.val_off[f], nv = a.in.val_off[f + 1] - v0;
    const uint32_t addr = (ot.flags & CL_OT_ADDR64) ? CL_TY_INT64 : CL_TY_INT32;
    const bool memop = ot.kind == CL_SK_LOAD || ot.kind == CL_SK_STORE || ot.kind == CL_SK_ATOMIC;
    const uint32_t n_slots = EXT ? total : 8u;
#define TS_FOR_SLOTS(s) _Pragma("unroll") for (uint32_t s = 0; s < n_slots; s++)
#define TS_TAG(s) (EXT ? (uint32_t)r.xt[s] : (uint32_t)r.tag8[s])
#define TS_PAY(s) (EXT ? r.xp[s] : r.pay8[s])

    /* operand-dependent parts of the signature */
    uint32_t loadw = 0, movlink = 0, elem = 0;
    const uint32_t accw = (mt.flags & CL_MT_F32) ? CL_TY_FLOAT32 : CL_TY_INT32;
    uint32_t role = CL_ROLE_SEED;
    switch (ot.kind) {
    case CL_SK_MOV: {                                                     /* typerec.py:135-139 */
        bool any_value = false, seen = false; uint32_t w = 1;
        TS_FOR_SLOTS(s) {
            if (s < u0 || s >= total) continue;
            const uint32_t t = TS_TAG(s);
            if (CL_T_KIND(t) == CL_K_VALUE) any_value = true;
            if (CL_T_KIND(t) == CL_K_CONSTMEM && !seen) { w = CL_T_WIDTH(t); seen = true; }
        }
        if (any_value) { loadw = movlink = TS_LINK; role = CL_ROLE_TRANSPARENT; } else loadw = ts_load_mask(w);
        break; }
    case CL_SK_LOAD: {                                                    /* :176-181 */
        uint32_t w = 1;
        TS_FOR_SLOTS(s) {
            if (s < d0 || s >= a0) continue;
            const uint32_t kd = CL_T_KIND(TS_TAG(s));
            if ((kd == CL_K_REG || kd == CL_K_UREG) && (TS_PAY(s) >> 16) > w) w = TS_PAY(s) >> 16;
        }
        if (CL_TH_DEFW(hint)) w = CL_TH_DEFW(hint);
        loadw = ts_load_mask(w);
        break; }
    case CL_SK_STORE: elem = (ot.flags & CL_OT_RED) ? mt.atom_elem : ts_load_mask(CL_TH_DATAW(hint) ? CL_TH_DATAW(hint) : 1u); break;
    case CL_SK_ATOMIC: elem = mt.atom_elem; break;
    case CL_SK_LOP: case CL_SK_SHF: case CL_SK_SHLR: case CL_SK_SEL: case CL_SK_SELECT: case CL_SK_PHI: case CL_SK_SHUFFLE:
        role = CL_ROLE_TRANSPARENT; break;
    case CL_SK_I2F: case CL_SK_F2I: case CL_SK_F2F: case CL_SK_I2I: case CL_SK_FRND: case CL_SK_CAST64: case CL_SK_BITCAST:
        role = CL_ROLE_CONVERSION; break;
    default: break;
    }

    uint32_t link_def = CL_NO_VALUE, link_mask = 0;
    TS_FOR_SLOTS(s) {
        if (s >= total) continue;
        const uint32_t t = TS_TAG(s), kd = CL_T_KIND(t);
        if (kd != CL_K_VALUE && kd != CL_K_MEMREF) continue;
        const uint32_t p = TS_PAY(s);
        if (s < d0) {                                                     /* guard, :334 */
            if (kd == CL_K_VALUE) ts_narrow(a, f, v0, nv, p, CL_TY_BOOL, false);
        } else if (s < a0) {                                              /* defs, :316-322 */
            if (kd != CL_K_VALUE) continue;
            const uint32_t c = ts_def_c(ot.kind, s - d0, mt, loadw, accw);
            if (c == TS_LINK) link_def = p;
            else if (c) ts_narrow(a, f, v0, nv, p, c, true);
        } else if (s < u0) {                                              /* aux defs, :323-325: Signature.aux is always Bool */
            if (kd == CL_K_VALUE) ts_narrow(a, f, v0, nv, p, CL_TY_BOOL, true);
        } else {                                                          /* uses, :326-333 */
            const uint32_t k = s - u0;
            const uint32_t c = (memop && kd == CL_K_MEMREF) ? addr : (ot.kind == CL_SK_LOAD) ? 0u
                               : ts_use_c(ot.kind, k, nu, ot, mt, movlink, elem, accw, hint);
            uint32_t ref = CL_NO_VALUE;
            if (kd == CL_K_VALUE) ref = p;
            else {
                const cl_memref m = a.in.mem[a.in.mem_off[f] + p];
                if (CL_T_KIND(m.base_tag) == CL_K_VALUE) ref = m.base_pay;
                if (CL_T_KIND(m.ureg_tag) == CL_K_VALUE) ts_narrow(a, f, v0, nv, m.ureg_pay, CL_TY_INT32, false);   /* _slot_values :281 */
            }
            if (ref == CL_NO_VALUE) continue;
            if (c == TS_LINK) link_mask |= 1u << (k < 15 ? k : 15);
            else if (c) ts_narrow(a, f, v0, nv, ref, c, false);
        }
    }
    a.role[i] = (uint8_t)role; a.link_mask[i] = (uint16_t)link_mask; a.link_def[i] = link_def;
#undef TS_FOR_SLOTS
#undef TS_TAG
#undef TS_PAY
}

TS_D void ts_record(const TsArgs &a, uint32_t i, uint32_t f) {
    TsRec r;
    const uint4 h4 = ((const uint4 *)a.in.hdr)[i];
    memcpy(&r.h, &h4, 16);
    r.f = f; r.g = (r.h.flags & CL_IF_GUARD) ? 1u : 0u;
    r.xt = nullptr; r.xp = nullptr;
    if (r.h.op >= a.n_ops || r.h.modset >= a.n_mods) { *a.bad = 1; a.role[i] = 0; a.link_mask[i] = 0; a.link_def[i] = CL_NO_VALUE; return; }
    if (r.h.flags & CL_IF_EXT) {
        r.xt = a.in.ext_tag + a.in.ext_off[f] + r.h.ext; r.xp = a.in.ext_pay + a.in.ext_off[f] + r.h.ext;
        ts_slots<true>(a, i, f, r);
    } else {
        const uint4 t4 = ((const uint4 *)a.in.tag)[i];
        const uint4 p0 = ((const uint4 *)a.in.pay)[2 * (size_t)i], p1 = ((const uint4 *)a.in.pay)[2 * (size_t)i + 1];
        memcpy(r.tag8, &t4, 16); memcpy(r.pay8, &p0, 16); memcpy(r.pay8 + 4, &p1, 16);
        ts_slots<false>(a, i, f, r);
    }
}

/* largest f with off[f] <= x */
TS_HD uint32_t ts_find(const uint32_t *off, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) { const uint32_t mid = (lo + hi) >> 1; if (off[mid] <= x) lo = mid; else hi = mid; }
    return lo;
}
/* a function may hold no record: skip to the one that owns record i */
TS_HD uint32_t ts_func_of(const uint32_t *rec_off, uint32_t F, uint32_t i) {
    uint32_t f = ts_find(rec_off, F, i);
    while (f + 1 < F && rec_off[f + 1] <= i) f++;
    return f;
}

TS_D void ts_block(const TsArgs &a, uint32_t b) {                         /* :342-343 */
    const cl_blk bl = a.in.blk[b];
    if (CL_T_KIND(bl.term_tag[0]) != CL_K_VALUE && CL_T_KIND(bl.term_tag[1]) != CL_K_VALUE) return;
    uint32_t f = ts_find(a.in.func_blk_off, a.in.n_funcs, b);
    while (f + 1 < a.in.n_funcs && a.in.func_blk_off[f + 1] <= b) f++;
    const uint32_t v0 = a.in.val_off[f], nv = a.in.val_off[f + 1] - v0;
    for (int t = 0; t < 2; t++)
        if (CL_T_KIND(bl.term_tag[t]) == CL_K_VALUE) ts_narrow(a, f, v0, nv, bl.term_pay[t], CL_TY_BOOL, false);
}

#if TS_CUDA
__global__ void __launch_bounds__(256) k_typeseed_prepare(TsArgs a, uint32_t *func_rec_off) {
    const size_t n = (size_t)gridDim.x * blockDim.x, t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (size_t v = t; v < a.n_val; v += n) a.val_masks[v] = 0xFFFFFFu;                 /* :292-295: TOP */
    for (size_t f = t; f <= a.in.n_funcs; f += n) {
        func_rec_off[f] = a.in.blk_off[a.in.func_blk_off[f]];
        if (f < a.in.n_funcs) a.status[f] = CL_ST_OK;
    }
}
__global__ void __launch_bounds__(256) k_typeseed(TsArgs a) {
    const uint32_t n = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
    for (uint32_t base = t - lane; base < a.n_inst; base += n) {
        /* one search per warp: the 32 records of a warp lie in a few neighbouring functions */
        uint32_t f = 0;
        if (lane == 0) f = ts_func_of(a.func_rec_off, a.in.n_funcs, base);
        f = __shfl_sync(0xFFFFFFFFu, f, 0);
        const uint32_t i = base + lane;
        if (i < a.n_inst) {
            while (f + 1 < a.in.n_funcs && a.func_rec_off[f + 1] <= i) f++;
            ts_record(a, i, f);
        }
    }
    for (uint32_t b = t; b < a.in.n_blocks; b += n) ts_block(a, b);
}
#define TS_OK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { rc = -1; snprintf(msg, sizeof msg, "%s: %s", #x, cudaGetErrorString(e_)); goto done; } } while (0)
#endif

extern "C" int cl_seed_types(cl_ctx *c, uint32_t source, const cl_optype *ops, uint32_t n_ops, const cl_modtype *mods, uint32_t n_mods,
                             const cl_typehints *hints, cl_typeseed *out) {
    TsArgs a{};
    void *stream_v = nullptr; float *last_ms = nullptr;
    uint64_t counts[2] = { 0, 0 };
    if (cli_corpus_view(c, source, &a.in, counts, &stream_v, &last_ms)) return -1;
    const uint32_t F = a.in.n_funcs, B = a.in.n_blocks;
    a.n_ops = n_ops; a.n_mods = n_mods;
    int rc = 0; char msg[400] = "";
#if TS_CUDA
    cudaStream_t st = (cudaStream_t)stream_v;
    uint8_t *blob = nullptr; cudaEvent_t e0 = nullptr, e1 = nullptr;
    {
        a.n_inst = (uint32_t)counts[0]; a.n_val = (uint32_t)counts[1];
        const size_t N = a.n_inst, V = a.n_val, H = hints ? hints->off[F] : 0;
        auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
        const size_t o_ops = 0, o_mods = o_ops + up(sizeof(cl_optype) * n_ops), o_hint = o_mods + up(sizeof(cl_modtype) * n_mods),
                     o_rec = o_hint + (hints ? up(4 * ((size_t)F + 1)) + 2 * up(4 * H) : 0), o_masks = o_rec + up(4 * ((size_t)F + 1)), o_role = o_masks + up(4 * V),
                     o_lm = o_role + up(N), o_ld = o_lm + up(2 * N), o_st = o_ld + up(4 * N), o_bad = o_st + up(F), total = o_bad + 256;
        TS_OK(cudaMalloc((void **)&blob, total));
        TS_OK(cudaMemcpyAsync(blob + o_ops, ops, sizeof(cl_optype) * n_ops, cudaMemcpyHostToDevice, st));
        TS_OK(cudaMemcpyAsync(blob + o_mods, mods, sizeof(cl_modtype) * n_mods, cudaMemcpyHostToDevice, st));
        if (hints) {
            uint8_t *h0 = blob + o_hint, *h1 = h0 + up(4 * ((size_t)F + 1)), *h2 = h1 + up(4 * H);
            TS_OK(cudaMemcpyAsync(h0, hints->off, 4 * ((size_t)F + 1), cudaMemcpyHostToDevice, st));
            if (H) { TS_OK(cudaMemcpyAsync(h1, hints->iid, 4 * H, cudaMemcpyHostToDevice, st)); TS_OK(cudaMemcpyAsync(h2, hints->val, 4 * H, cudaMemcpyHostToDevice, st)); }
            a.hint_off = (const uint32_t *)h0; a.hint_iid = (const uint32_t *)h1; a.hint_val = (const uint32_t *)h2;
        }
        TS_OK(cudaMemsetAsync(blob + o_bad, 0, 4, st));
        a.ops = (const cl_optype *)(blob + o_ops); a.mods = (const cl_modtype *)(blob + o_mods);
        a.func_rec_off = (const uint32_t *)(blob + o_rec);
        a.val_masks = (uint32_t *)(blob + o_masks); a.role = blob + o_role; a.link_mask = (uint16_t *)(blob + o_lm);
        a.link_def = (uint32_t *)(blob + o_ld); a.status = blob + o_st; a.bad = (uint32_t *)(blob + o_bad);
        int dev = 0, n_sm = 148;
        cudaGetDevice(&dev); cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        const unsigned grid = (unsigned)n_sm * 8;             /* 8 CTAs of 256 threads per SM: full occupancy, grid-stride */
        TS_OK(cudaEventCreate(&e0)); TS_OK(cudaEventCreate(&e1));
        TS_OK(cudaEventRecord(e0, st));
        k_typeseed_prepare<<<grid, 256, 0, st>>>(a, (uint32_t *)(blob + o_rec));
        k_typeseed<<<grid, 256, 0, st>>>(a);
        TS_OK(cudaGetLastError());
        TS_OK(cudaEventRecord(e1, st));
        uint32_t bad = 0;
        TS_OK(cudaMemcpyAsync(out->val_masks, a.val_masks, 4 * V, cudaMemcpyDeviceToHost, st));
        TS_OK(cudaMemcpyAsync(out->role, a.role, N, cudaMemcpyDeviceToHost, st));
        TS_OK(cudaMemcpyAsync(out->link_mask, a.link_mask, 2 * N, cudaMemcpyDeviceToHost, st));
        TS_OK(cudaMemcpyAsync(out->link_def, a.link_def, 4 * N, cudaMemcpyDeviceToHost, st));
        TS_OK(cudaMemcpyAsync(out->status, a.status, F, cudaMemcpyDeviceToHost, st));
        TS_OK(cudaMemcpyAsync(&bad, a.bad, 4, cudaMemcpyDeviceToHost, st));
        TS_OK(cudaStreamSynchronize(st));
        if (last_ms) TS_OK(cudaEventElapsedTime(last_ms, e0, e1));
        if (bad) { rc = -1; snprintf(msg, sizeof msg, "cl_seed_types: opcode / modset id outside the tables"); }
    }
done:
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (blob) cudaFree(blob);
#else
    (void)stream_v;
    a.n_inst = (uint32_t)counts[0]; a.n_val = (uint32_t)counts[1];
    a.ops = ops; a.mods = mods;
    if (hints) { a.hint_off = hints->off; a.hint_iid = hints->iid; a.hint_val = hints->val; }
    uint32_t *rec_off = (uint32_t *)malloc(4 * ((size_t)F + 1)), bad = 0;
    for (uint32_t f = 0; f <= F; f++) rec_off[f] = a.in.blk_off[a.in.func_blk_off[f]];
    a.func_rec_off = rec_off;
    a.val_masks = out->val_masks; a.role = out->role; a.link_mask = out->link_mask; a.link_def = out->link_def; a.status = out->status; a.bad = &bad;
    for (uint32_t v = 0; v < a.n_val; v++) a.val_masks[v] = 0xFFFFFFu;
    for (uint32_t f = 0; f < F; f++) a.status[f] = CL_ST_OK;
    for (uint32_t i = 0; i < a.n_inst; i++) ts_record(a, i, ts_func_of(rec_off, F, i));
    for (uint32_t b = 0; b < B; b++) ts_block(a, b);
    free(rec_off);
    if (last_ms) *last_ms = 0;
    if (bad) { rc = -1; snprintf(msg, sizeof msg, "cl_seed_types: opcode / modset id outside the tables"); }
#endif
    if (rc) { cli_set_error(msg); return -1; }
    return 0;
}

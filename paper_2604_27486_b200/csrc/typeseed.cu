/* typeseed.cu -- cl_seed_types of include/culifter_types.h on sm_100a:
 * typerec.seed_types (reference typerec.py:288-345) with signature_for
 * (typerec.py:78-235) evaluated per record on the device.
 *
 * Four launches on the context's stream:
 *   k_typeseed_prepare  every value word at TOP (dead vids carry a marker), first record of every function
 *   k_typeseed_index    function of every run of 32 records (one binary search per run, all in parallel)
 *   k_typeseed          one thread per instruction record (grid-stride, 148 SMs x 8 CTAs of 256): the three planes
 *                       of a record are read once with 128-bit loads (64 B) and stay in registers; the constraint
 *                       of a def / aux def / use slot is a cell of a 51-row signature table in shared memory (the
 *                       reference's if-chain evaluated once on the host: literal mask, LINK, or a per-record
 *                       parameter such as the element type of the modifier tuple); every constrained value is
 *                       narrowed with ONE 32-bit red.and on its packed word (seed | def << 8 | use << 16), so the
 *                       order of the records does not matter; 7 bytes written per record (role, link mask, link
 *                       def); then one thread per function narrows the terminator conditions of its blocks
 *   k_typeseed_check    a dead vid whose word moved was narrowed: KeyError upstream; dead words read TOP again
 * HBM bound in principle: 64 B read + 7 B written per record + 8 B per value; measured 34 % of the HBM roofline,
 * DRAM traffic 1.04 x the algorithmic bytes (profiles/r02_tuning.md).
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
#define TS_TOP3 0xFFFFFFu        /* seed | def << 8 | use << 16, all at top */
#define TS_DEAD 0x80000000u      /* fill marker of a vid that is not in fn.values */

struct TsArgs {
    cl_corpus in;                    /* device pointers */
    const uint32_t *func_rec_off;    /* [F+1] first record of every function */
    const uint32_t *warp_func;       /* [ceil(n_inst / 32)] function of the first record of every run of 32 records */
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
    /* a value that is not in fn.values (KeyError upstream): its word carries TS_DEAD from the fill, any narrowing of it
     * is found by the check pass -- no load of val_alive in front of every red.and                                   */
    if (vid >= nv) { a.status[f] = CL_ST_KEY_ERROR; return; }
    const uint32_t drop = ~mask & 0xFFu;
    if (drop) ts_and(a.val_masks + v0 + vid, ~(drop | (is_def ? drop << 8 : drop << 16)));
}

/* ------------------------------------------------------------------ signature table
 * The two switches above are evaluated ONCE on the host into a table the kernel indexes (a switch per slot made
 * the lanes of a warp, which hold 32 different opcodes, run one after the other: 8 of 32 lanes active).  A row is a
 * signature kind, or one of five variants picked by the modifier tuple / the operands; a cell is a literal mask,
 * TS_LINK, or a sentinel naming a per-record parameter (element type of the modifier tuple, load width ...).   */
enum { TS_ROW_IMAD_WIDE = CL_SK__COUNT, TS_ROW_LEA_HI, TS_ROW_BITCAST_F2I, TS_ROW_BITCAST_I2F, TS_ROW_MOV_LINK, TS_ROWS };
enum { TS_P_F16 = 0xE1, TS_P_MMA, TS_P_CONVF, TS_P_CONVI, TS_P_F2FD, TS_P_F2FS, TS_P_ATOM, TS_P_LOADW, TS_P_ELEM, TS_P_ACCW };
struct TsRow { uint16_t cell[10]; uint16_t role, pad; };      /* cell[0..1]: defs k = 0, k >= 1; cell[2..9]: uses k = 0..6, k >= 7 */

static void ts_build_table(TsRow *tab) {
    cl_modtype mt; mt.f16_elem = TS_P_F16; mt.mma_elem = TS_P_MMA; mt.conv_float = TS_P_CONVF; mt.conv_int = TS_P_CONVI;
    mt.f2f_dst = TS_P_F2FD; mt.f2f_src = TS_P_F2FS; mt.atom_elem = TS_P_ATOM; mt.flags = 0;
    const cl_optype ot = { 0, 0 };
    for (uint32_t row = 0; row < TS_ROWS; row++) {
        uint32_t kind = row, movlink = 0, loadw = TS_P_LOADW;
        cl_modtype m = mt;
        switch (row) {
        case TS_ROW_IMAD_WIDE: kind = CL_SK_IMAD; m.flags = CL_MT_WIDE; break;
        case TS_ROW_LEA_HI: kind = CL_SK_LEA; m.flags = CL_MT_HI; break;
        case TS_ROW_BITCAST_F2I: kind = CL_SK_BITCAST; m.flags = CL_MT_F2I; break;
        case TS_ROW_BITCAST_I2F: kind = CL_SK_BITCAST; m.flags = CL_MT_I2F; break;
        case TS_ROW_MOV_LINK: kind = CL_SK_MOV; movlink = TS_LINK; loadw = TS_LINK; break;
        default: break;
        }
        for (uint32_t k = 0; k < 2; k++) tab[row].cell[k] = (uint16_t)ts_def_c(kind, k, m, loadw, TS_P_ACCW);
        for (uint32_t k = 0; k < 8; k++) tab[row].cell[2 + k] = (uint16_t)ts_use_c(kind, k, 255, ot, m, movlink, TS_P_ELEM, TS_P_ACCW, 0);
        uint32_t role = CL_ROLE_SEED;
        switch (kind) {
        case CL_SK_LOP: case CL_SK_SHF: case CL_SK_SHLR: case CL_SK_SEL: case CL_SK_SELECT: case CL_SK_PHI: case CL_SK_SHUFFLE:
            role = CL_ROLE_TRANSPARENT; break;
        case CL_SK_I2F: case CL_SK_F2I: case CL_SK_F2F: case CL_SK_I2I: case CL_SK_FRND: case CL_SK_CAST64: case CL_SK_BITCAST:
            role = CL_ROLE_CONVERSION; break;
        default: break;
        }
        if (row == TS_ROW_MOV_LINK) role = CL_ROLE_TRANSPARENT;
        tab[row].role = (uint16_t)role; tab[row].pad = 0;
    }
}

/* a table cell with its parameter resolved: p0 / p1 hold the ten per-record parameters, one byte each */
TS_HD uint32_t ts_cell(uint32_t c, uint64_t p0, uint32_t p1) {
    const uint32_t i = c - TS_P_F16;
    if (i >= 10u) return c;
    return i < 8u ? (uint32_t)(p0 >> (8u * i)) & 0xFFu : (p1 >> (8u * (i - 8u))) & 0xFFu;
}

/* One record.  EXT = false: the 8 inline slots sit in registers and every slot loop is unrolled over the absolute
 * slot index (no local-memory array); EXT = true (more than 8 slots: wide PHIs, tensor ops): slots are read from
 * the function's overflow region.                                                                              */
template <bool EXT> TS_D void ts_slots(const TsArgs &a, const TsRow *tab, uint32_t i, uint32_t f, const TsRec &r) {
    const cl_optype ot = a.ops[r.h.op];
    const cl_modtype mt = a.mods[r.h.modset];
    const uint32_t kind = ot.kind;
    const bool is_load = kind == CL_SK_LOAD, is_store = kind == CL_SK_STORE, is_tensor = kind == CL_SK_TENSOR;
    /* only loads, stores and tensor ops read Instruction.meta */
    const uint32_t hint = (a.hint_off && (is_load || is_store || is_tensor)) ? ts_hint(a, f, r.h.iid) : 0u;
    const uint32_t nd = r.h.n_defs, na = r.h.n_aux, nu = r.h.n_uses;
    const uint32_t d0 = r.g, a0 = d0 + nd, u0 = a0 + na, total = u0 + nu;
    const uint32_t v0 = a.in.val_off[f], nv = a.in.val_off[f + 1] - v0;
    const uint32_t addr = (ot.flags & CL_OT_ADDR64) ? CL_TY_INT64 : CL_TY_INT32;
    const bool memop = is_load || is_store || kind == CL_SK_ATOMIC;
    const uint32_t n_slots = EXT ? total : 8u;
#define TS_FOR_SLOTS(s) _Pragma("unroll") for (uint32_t s = 0; s < n_slots; s++)
#define TS_TAG(s) (EXT ? (uint32_t)r.xt[s] : (uint32_t)r.tag8[s])
#define TS_PAY(s) (EXT ? r.xp[s] : r.pay8[s])

    /* operand-dependent parts of the signature: is a use of a MOV a value, width of its first ConstMem use
     * (typerec.py:135-139); widest Reg / UReg def of a load (:176-181).  Two short loops that only the lanes holding a
     * MOV / a load run (one loop over all slots for every record cost 17 % of the kernel's instructions).          */
    bool any_value = false; uint32_t cmw = 1, regw = 1;
    if (kind == CL_SK_MOV) {
        bool seen = false;
        TS_FOR_SLOTS(s) {
            const uint32_t t = TS_TAG(s), kd = CL_T_KIND(t);
            const bool is_use = s >= u0 && s < total;
            any_value |= is_use && kd == CL_K_VALUE;
            if (is_use && kd == CL_K_CONSTMEM && !seen) { cmw = CL_T_WIDTH(t); seen = true; }
        }
    } else if (is_load) {
        TS_FOR_SLOTS(s) {
            const uint32_t kd = CL_T_KIND(TS_TAG(s)), w = TS_PAY(s) >> 16;
            if (s >= d0 && s < a0 && (kd == CL_K_REG || kd == CL_K_UREG) && w > regw) regw = w;
        }
    }
    const uint32_t loadw = ts_load_mask(is_load ? (CL_TH_DEFW(hint) ? CL_TH_DEFW(hint) : regw) : cmw);
    const uint32_t elem = (is_store && !(ot.flags & CL_OT_RED)) ? ts_load_mask(CL_TH_DATAW(hint) ? CL_TH_DATAW(hint) : 1u) : mt.atom_elem;
    const uint32_t accw = (mt.flags & CL_MT_F32) ? CL_TY_FLOAT32 : CL_TY_INT32;
    const uint64_t p0 = (uint64_t)mt.f16_elem | (uint64_t)mt.mma_elem << 8 | (uint64_t)mt.conv_float << 16 | (uint64_t)mt.conv_int << 24
                        | (uint64_t)mt.f2f_dst << 32 | (uint64_t)mt.f2f_src << 40 | (uint64_t)mt.atom_elem << 48 | (uint64_t)loadw << 56;
    const uint32_t p1 = elem | accw << 8;
    uint32_t row = kind;
    row = (kind == CL_SK_IMAD && (mt.flags & CL_MT_WIDE)) ? (uint32_t)TS_ROW_IMAD_WIDE : row;
    row = (kind == CL_SK_LEA && (mt.flags & CL_MT_HI)) ? (uint32_t)TS_ROW_LEA_HI : row;
    row = (kind == CL_SK_BITCAST && (mt.flags & CL_MT_I2F)) ? (uint32_t)TS_ROW_BITCAST_I2F : row;
    row = (kind == CL_SK_BITCAST && (mt.flags & CL_MT_F2I)) ? (uint32_t)TS_ROW_BITCAST_F2I : row;     /* F2I is tested first (:170) */
    row = (kind == CL_SK_MOV && any_value) ? (uint32_t)TS_ROW_MOV_LINK : row;
    const TsRow &sig = tab[row < (uint32_t)TS_ROWS ? row : 0u];
    const uint32_t n_ab = CL_TH_NA(hint) + CL_TH_NB(hint), n_abc = n_ab + CL_TH_NC(hint);      /* tensor operand groups, :209-214 */

    uint32_t link_def = CL_NO_VALUE, link_mask = 0;
    TS_FOR_SLOTS(s) {
        if (s >= total) continue;
        const uint32_t t = TS_TAG(s), kd = CL_T_KIND(t);
        if (kd != CL_K_VALUE && kd != CL_K_MEMREF) continue;
        const uint32_t p = TS_PAY(s);
        const bool is_use = s >= u0, is_defslot = s >= d0 && s < a0, is_memref = kd == CL_K_MEMREF;
        if (!is_use && is_memref) continue;                               /* defs, aux defs and the guard: values only */
        const uint32_t k = is_use ? s - u0 : s - d0;
        /* the constraint: Bool for the guard (:334) and the aux defs (:323-325), else the table cell */
        uint32_t c = sig.cell[is_use ? 2u + (EXT ? (k < 7u ? k : 7u) : k) : (k ? 1u : 0u)];
        if (is_use && is_tensor) c = k < n_ab ? (uint32_t)TS_P_MMA : k < n_abc ? (uint32_t)TS_P_ACCW : 0u;
        c = ts_cell(c, p0, p1);
        if (is_use && memop && is_memref) c = addr;
        if (!is_use && !is_defslot) c = CL_TY_BOOL;
        uint32_t ref = p;
        if (is_memref) {                                                  /* _slot_values, :273-284 */
            const cl_memref m = a.in.mem[a.in.mem_off[f] + p];
            ref = CL_T_KIND(m.base_tag) == CL_K_VALUE ? m.base_pay : CL_NO_VALUE;
            if (CL_T_KIND(m.ureg_tag) == CL_K_VALUE) ts_narrow(a, f, v0, nv, m.ureg_pay, CL_TY_INT32, false);
            if (ref == CL_NO_VALUE) continue;
        }
        const bool link = c == TS_LINK;                                   /* LINK cells: bookkeeping without a branch */
        link_mask |= (link && is_use) ? 1u << (EXT ? (k < 15u ? k : 15u) : k) : 0u;
        link_def = (link && !is_use) ? p : link_def;
        if (!link && c) ts_narrow(a, f, v0, nv, ref, c, !is_use && s >= d0);
    }
    a.role[i] = (uint8_t)sig.role; a.link_mask[i] = (uint16_t)link_mask; a.link_def[i] = link_def;
#undef TS_FOR_SLOTS
#undef TS_TAG
#undef TS_PAY
}

/* the 64 bytes of a record as four 128-bit words (header, tags, payloads) */
struct TsPlanes { uint4 h, t, p0, p1; };
TS_D TsPlanes ts_load(const TsArgs &a, uint32_t i) {
    TsPlanes q;
    q.h = ((const uint4 *)a.in.hdr)[i]; q.t = ((const uint4 *)a.in.tag)[i];
    q.p0 = ((const uint4 *)a.in.pay)[2 * (size_t)i]; q.p1 = ((const uint4 *)a.in.pay)[2 * (size_t)i + 1];
    return q;
}
TS_D void ts_record(const TsArgs &a, const TsRow *tab, uint32_t i, uint32_t f, const TsPlanes &q) {
    TsRec r;
    memcpy(&r.h, &q.h, 16);
    r.f = f; r.g = (r.h.flags & CL_IF_GUARD) ? 1u : 0u;
    r.xt = nullptr; r.xp = nullptr;
    if (r.h.op >= a.n_ops || r.h.modset >= a.n_mods) { *a.bad = 1; a.role[i] = 0; a.link_mask[i] = 0; a.link_def[i] = CL_NO_VALUE; return; }
    if (r.h.flags & CL_IF_EXT) {
        r.xt = a.in.ext_tag + a.in.ext_off[f] + r.h.ext; r.xp = a.in.ext_pay + a.in.ext_off[f] + r.h.ext;
        ts_slots<true>(a, tab, i, f, r);
    } else {
        memcpy(r.tag8, &q.t, 16); memcpy(r.pay8, &q.p0, 16); memcpy(r.pay8 + 4, &q.p1, 16);
        ts_slots<false>(a, tab, i, f, r);
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

TS_D void ts_block(const TsArgs &a, uint32_t b, uint32_t f) {             /* :342-343 */
    const cl_blk bl = a.in.blk[b];
    const uint32_t v0 = a.in.val_off[f], nv = a.in.val_off[f + 1] - v0;
    for (int t = 0; t < 2; t++)
        if (CL_T_KIND(bl.term_tag[t]) == CL_K_VALUE) ts_narrow(a, f, v0, nv, bl.term_pay[t], CL_TY_BOOL, false);
}
/* after the narrowing: a dead vid whose word moved was narrowed (KeyError upstream); dead words read TOP again */
TS_D void ts_check_value(const TsArgs &a, uint32_t v) {
    const uint32_t m = a.val_masks[v];
    if (!(m & TS_DEAD)) return;
    if (m != (TS_DEAD | TS_TOP3)) a.status[ts_func_of(a.in.val_off, a.in.n_funcs, v)] = CL_ST_KEY_ERROR;
    a.val_masks[v] = TS_TOP3;
}

#if TS_CUDA
__global__ void __launch_bounds__(256) k_typeseed_prepare(TsArgs a, uint32_t *func_rec_off) {
    const size_t n = (size_t)gridDim.x * blockDim.x, t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    /* :292-295: every value at TOP; four values per thread (the arrays start 256-byte aligned) */
    const size_t quads = a.n_val / 4;
    for (size_t q = t; q < quads; q += n) {
        const uint32_t al = ((const uint32_t *)a.in.val_alive)[q];
        uint4 m;
        m.x = (al & 0xFFu) ? TS_TOP3 : (TS_DEAD | TS_TOP3); m.y = (al & 0xFF00u) ? TS_TOP3 : (TS_DEAD | TS_TOP3);
        m.z = (al & 0xFF0000u) ? TS_TOP3 : (TS_DEAD | TS_TOP3); m.w = (al & 0xFF000000u) ? TS_TOP3 : (TS_DEAD | TS_TOP3);
        ((uint4 *)a.val_masks)[q] = m;
    }
    for (size_t v = quads * 4 + t; v < a.n_val; v += n) a.val_masks[v] = a.in.val_alive[v] ? TS_TOP3 : (TS_DEAD | TS_TOP3);
    for (size_t f = t; f <= a.in.n_funcs; f += n) {
        func_rec_off[f] = a.in.blk_off[a.in.func_blk_off[f]];
        if (f < a.in.n_funcs) a.status[f] = CL_ST_OK;
    }
}
/* one binary search per run of 32 records, all in parallel (the record kernel used to search with lane 0 of every
 * warp while 31 lanes waited: 30 % of its stall samples)                                                        */
__global__ void __launch_bounds__(256) k_typeseed_index(TsArgs a, uint32_t *warp_func) {
    const uint32_t n = gridDim.x * blockDim.x, n_runs = (a.n_inst + 31) / 32;
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n_runs; w += n) warp_func[w] = ts_func_of(a.func_rec_off, a.in.n_funcs, w * 32);
}
#ifndef TS_MINB
#define TS_MINB 5          /* resident CTAs per SM asked of ptxas: 45 registers, no spill (4 / 5 / 6 / 8 measured alike) */
#endif
__global__ void __launch_bounds__(256, TS_MINB) k_typeseed(TsArgs a, const TsRow *g_tab) {
    __shared__ TsRow tab[TS_ROWS];
    for (uint32_t w = threadIdx.x; w < sizeof(tab) / 4; w += blockDim.x) ((uint32_t *)tab)[w] = ((const uint32_t *)g_tab)[w];
    __syncthreads();
    const uint32_t n = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x;
    /* (requesting the planes of the thread's next record before working on the current one was measured: no gain,
     * 0.904 vs 0.903 ms, and 63 registers instead of 45) */
    for (uint32_t i = t; i < a.n_inst; i += n) {
        uint32_t f = a.warp_func[i >> 5];                     /* the 32 records of a warp lie in a few neighbouring functions */
        while (f + 1 < a.in.n_funcs && a.func_rec_off[f + 1] <= i) f++;
        ts_record(a, tab, i, f, ts_load(a, i));
    }
    for (uint32_t f = t; f < a.in.n_funcs; f += n)            /* terminator conditions of the function's blocks */
        for (uint32_t b = a.in.func_blk_off[f]; b < a.in.func_blk_off[f + 1]; b++) ts_block(a, b, f);
}
__global__ void __launch_bounds__(256) k_typeseed_check(TsArgs a) {
    const uint32_t n = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x, quads = a.n_val / 4;
    for (uint32_t q = t; q < quads; q += n) {
        const uint4 m = ((const uint4 *)a.val_masks)[q];
        if ((m.x | m.y | m.z | m.w) & TS_DEAD)
            for (uint32_t v = 4 * q; v < 4 * q + 4; v++) ts_check_value(a, v);
    }
    for (uint32_t v = quads * 4 + t; v < a.n_val; v += n) ts_check_value(a, v);
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
    (void)B;
    a.n_ops = n_ops; a.n_mods = n_mods;
    int rc = 0; char msg[400] = "";
    static TsRow h_tab[TS_ROWS];
    ts_build_table(h_tab);
#if TS_CUDA
    cudaStream_t st = (cudaStream_t)stream_v;
    uint8_t *blob = nullptr; cudaEvent_t e0 = nullptr, e1 = nullptr;
    {
        a.n_inst = (uint32_t)counts[0]; a.n_val = (uint32_t)counts[1];
        const size_t N = a.n_inst, V = a.n_val, H = hints ? hints->off[F] : 0;
        auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
        const size_t o_ops = 0, o_mods = o_ops + up(sizeof(cl_optype) * n_ops), o_hint = o_mods + up(sizeof(cl_modtype) * n_mods),
                     o_rec = o_hint + (hints ? up(4 * ((size_t)F + 1)) + 2 * up(4 * H) : 0), o_masks = o_rec + up(4 * ((size_t)F + 1)), o_role = o_masks + up(4 * V),
                     o_lm = o_role + up(N), o_ld = o_lm + up(2 * N), o_st = o_ld + up(4 * N), o_bad = o_st + up(F), o_tab = o_bad + 256, o_wf = o_tab + up(sizeof(TsRow) * TS_ROWS), total = o_wf + up(4 * ((N + 31) / 32 + 1));
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
        TS_OK(cudaMemcpyAsync(blob + o_tab, h_tab, sizeof(TsRow) * TS_ROWS, cudaMemcpyHostToDevice, st));
        a.ops = (const cl_optype *)(blob + o_ops); a.mods = (const cl_modtype *)(blob + o_mods);
        a.func_rec_off = (const uint32_t *)(blob + o_rec); a.warp_func = (const uint32_t *)(blob + o_wf);
        a.val_masks = (uint32_t *)(blob + o_masks); a.role = blob + o_role; a.link_mask = (uint16_t *)(blob + o_lm);
        a.link_def = (uint32_t *)(blob + o_ld); a.status = blob + o_st; a.bad = (uint32_t *)(blob + o_bad);
        int dev = 0, n_sm = 148;
        cudaGetDevice(&dev); cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        const unsigned grid = (unsigned)n_sm * 8;             /* 8 CTAs of 256 threads per SM: full occupancy, grid-stride */
        TS_OK(cudaEventCreate(&e0)); TS_OK(cudaEventCreate(&e1));
        TS_OK(cudaEventRecord(e0, st));
        k_typeseed_prepare<<<grid, 256, 0, st>>>(a, (uint32_t *)(blob + o_rec));
        k_typeseed_index<<<grid, 256, 0, st>>>(a, (uint32_t *)(blob + o_wf));
        k_typeseed<<<grid, 256, 0, st>>>(a, (const TsRow *)(blob + o_tab));
        k_typeseed_check<<<grid, 256, 0, st>>>(a);
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
    for (uint32_t v = 0; v < a.n_val; v++) a.val_masks[v] = a.in.val_alive[v] ? TS_TOP3 : (TS_DEAD | TS_TOP3);
    for (uint32_t f = 0; f < F; f++) a.status[f] = CL_ST_OK;
    for (uint32_t i = 0; i < a.n_inst; i++) ts_record(a, h_tab, i, ts_func_of(rec_off, F, i), ts_load(a, i));
    for (uint32_t f = 0; f < F; f++)
        for (uint32_t b = a.in.func_blk_off[f]; b < a.in.func_blk_off[f + 1]; b++) ts_block(a, b, f);
    for (uint32_t v = 0; v < a.n_val; v++) ts_check_value(a, v);
    free(rec_off);
    if (last_ms) *last_ms = 0;
    if (bad) { rc = -1; snprintf(msg, sizeof msg, "cl_seed_types: opcode / modset id outside the tables"); }
#endif
    if (rc) { cli_set_error(msg); return -1; }
    return 0;
}

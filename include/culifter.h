/* culifter.h -- C ABI and struct-of-arrays layout of the B200 normalisation +
 * pattern-aggregation path (the data-parallel core of CuLifter / sasslift).
 *
 * Two shared libraries implement this header with identical semantics:
 *   paper_2604_27486_b200/csrc/libculifter.so   the product: sm_100a CUDA kernels
 *   oracle/liboracle.so                         TEST INFRASTRUCTURE: sequential C
 *                                               restatement of the reference
 * Every entry point cites the reference interface it replaces (paths relative
 * to /root/reference/pkg/src/sasslift/).
 *
 * ------------------------------------------------------------------------
 * Instruction stream layout ("SoA corpus")
 * ------------------------------------------------------------------------
 * A corpus is F independent functions (LiftedFunction, ssir.py:203).  A
 * function owns a sorted run of basic blocks (block_order(), ssir.py:244) and
 * each block owns a contiguous run of instruction records.  An instruction is
 * three planes, 64 bytes in total:
 *
 *   hdr  cl_hdr            16 B   iid, opcode id, modifier-set id, arities, flags
 *   tag  uint16_t[8]       16 B   operand kind + syntactic flags per slot
 *   pay  uint32_t[8]       32 B   operand payload per slot
 *
 * Slots are packed in the order  [guard] defs aux_defs uses  (Instruction,
 * ssir.py:42-51).  When 1*has_guard + n_defs + n_aux + n_uses > 8 the record
 * has CL_IF_EXT set and *all* slots live in the function's ext_tag/ext_pay
 * region starting at hdr.ext (PHI with many inputs, tensor ops).
 *
 * All indices stored inside a function (vid, imm index, memref index, ext
 * offset) are function-local, so a function region can be relocated freely;
 * that is what lets the corpus be sharded by function across GPUs with no
 * fix-up.
 *
 * At the ABI boundary every stream is a dense CSR (offset arrays of length
 * n+1).  On the device every function's result is written once, at an
 * atomically reserved place (completion order); the run densifies it to
 * function order on the device as its last step, so cl_download() is a plain
 * D2H copy (it overlaps the kernels of other contexts: capi.Pipeline).
 */
#ifndef CULIFTER_H
#define CULIFTER_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ opcodes */
#define CL_OPF_PURE   1u
#define CL_OPF_LDST   2u
#define CL_OPF_GLOBAL 4u
#define CL_OPF_ATOMIC 8u
#define CL_OPF_LOAD   16u
#define CL_OPF_D64    32u

enum cl_opcode {
#define CL_OP(name, flags) CL_OP_##name,
#include "culifter_ops.h"
#undef CL_OP
    CL_OP__COUNT
};

/* ------------------------------------------------------------ operand slots */
/* tag bits: kind[0:4) neg[4] not[5] abs[6] half[7:9) reuse[9] width[10:13)
 * bits 13..15 are kind specific (immediates, below).                        */
enum cl_kind {
    CL_K_NONE = 0,
    CL_K_VALUE = 1,    /* ValueRef  pay = vid                                  */
    CL_K_IMM = 2,      /* Imm       pay = function-local index into imm table  */
    CL_K_RZ = 3,       /* ZeroReg(uniform=False)                               */
    CL_K_URZ = 4,      /* ZeroReg(uniform=True)                                */
    CL_K_PRED = 5,     /* Pred      pay = index (7 = PT)                       */
    CL_K_REG = 6,      /* Reg       pay = base | width << 16                   */
    CL_K_UREG = 7,     /* UReg      pay = index | width << 16                  */
    CL_K_CONSTMEM = 8, /* ConstMem  pay = offset | bank << 20, width in tag    */
    CL_K_SREG = 9,     /* SReg      pay = host string id                       */
    CL_K_MEMREF = 10   /* MemRef    pay = function-local index into memrefs    */
};
#define CL_T_KIND(t)    ((t) & 15u)
#define CL_T_NEG        (1u << 4)
#define CL_T_NOT        (1u << 5)
#define CL_T_ABS        (1u << 6)
#define CL_T_HALF(t)    (((t) >> 7) & 3u)   /* 0 none, 1 H0, 2 H1 */
#define CL_T_HALF_SHIFT 7
#define CL_T_REUSE      (1u << 9)
#define CL_T_WIDTH(t)   (((t) >> 10) & 7u)
#define CL_T_WIDTH_SHIFT 10
/* immediates reuse the flag bits: NEG = Imm.negated, NOT = Imm.is_float,
 * ABS = text is "hex(cl_imm.text)" instead of host string id cl_imm.text      */
#define CL_T_IMM_FLOAT   CL_T_NOT
#define CL_T_IMM_HEXTEXT CL_T_ABS
#define CL_PT_INDEX 7u
#define CL_CM_OFFSET_BITS 20
#define CL_CM_PAY(bank, off) (((uint32_t)(bank) << CL_CM_OFFSET_BITS) | (uint32_t)(off))

typedef struct cl_hdr {
    uint32_t iid;
    uint16_t op;        /* enum cl_opcode or dynamic id >= CL_OP__COUNT         */
    uint16_t modset;    /* interned ordered modifier tuple (cl_modset table)     */
    uint8_t n_defs, n_aux, n_uses;
    uint8_t flags;      /* CL_IF_*                                              */
    uint32_t ext;       /* function-local offset into ext_* when CL_IF_EXT;
                           else, when CL_IF_SYNTH: iid of the instruction whose
                           source line (`raw`) the synthetic one shares          */
} cl_hdr;

#define CL_IF_EXT      0x01u  /* slots live in the ext region                    */
#define CL_IF_GUARD    0x02u  /* slot 0 is the guard predicate                   */
#define CL_IF_SYNTH    0x04u  /* meta["synthetic"] (x4-scale / sr-substitute)    */
/* tag_cuda_objects (patterns.py:895): object kind + which use carries the id */
#define CL_IF_OBJ_SHIFT 3
#define CL_IF_OBJ_MASK  (3u << CL_IF_OBJ_SHIFT)  /* 1 block_sync 2 warp_group 3 collective */
#define CL_IF_OBJUSE_SHIFT 5                      /* use index 0..6, 7 = none    */
#define CL_IF_OBJUSE_MASK (7u << CL_IF_OBJUSE_SHIFT)

typedef struct cl_imm {     /* Imm (operands.py:161): 64-bit pattern + spelling  */
    uint64_t bits;
    uint64_t text;          /* host string id, or the value whose hex() is shown */
} cl_imm;

typedef struct cl_memref {  /* MemRef (operands.py:213)                          */
    uint16_t base_tag, ureg_tag;
    uint32_t base_pay, ureg_pay;
    int32_t off_hi;         /* offset = off_hi:off_lo as a signed 64-bit         */
    uint32_t off_lo;
} cl_memref;

typedef struct cl_blk {     /* BasicBlock (ssir.py:174) + terminator value uses  */
    uint32_t bid;
    uint16_t term_tag[2];   /* cond, guard of CondBr/CondExit (ssir.py:378)      */
    uint32_t term_pay[2];
} cl_blk;

enum cl_arch { CL_ARCH_SM52 = 0, CL_ARCH_SM75, CL_ARCH_SM90, CL_ARCH_SM100, CL_ARCH_SM120 };

/* per-function status written by the passes */
enum cl_status {
    CL_ST_OK = 0,
    CL_ST_CAPACITY = 1,       /* an output region was too small: re-run with more  */
    CL_ST_ATTRIBUTE_ERROR = 2,/* reference raises AttributeError (non-value def)   */
    CL_ST_ASSERTION_ERROR = 3,/* reference _var_operand assertion (patterns.py:524)*/
    CL_ST_KEY_ERROR = 4,      /* reference KeyError (patterns.py:885, :310)        */
    CL_ST_UNSUPPORTED = 5,    /* shape outside this implementation: loud failure   */
    CL_ST_INDEX_ERROR = 6     /* reference IndexError (e.g. MUFU.RCP without a def) */
};
/* A function whose status is not CL_ST_OK is returned UNCHANGED (its input
 * stream, value table and counters): the reference reports such a function as
 * a per-function error (pipeline.py:182-188) and its partial state is unused. */

typedef struct cl_func {    /* LiftedFunction counters (ssir.py:215-217)         */
    uint32_t next_vid, next_iid, next_temp_reg;
    uint8_t arch, status;
    uint16_t reserved;
} cl_func;

/* modifier-set side table, computed by the host for the current pattern table:
 * one bit per modifier of the "universe" (built-ins below + every modifier a
 * pattern mentions).                                                          */
enum cl_modbit { CL_MB_X4 = 0, CL_MB_WIDE, CL_MB_U32, CL_MB_S32, CL_MB_LO, CL_MB_HI,
                 CL_MB_RCP, CL_MB_SYNC, CL_MB_64, CL_MB_128, CL_MB_F64, CL_MB_S64,
                 CL_MB_U64, CL_MB__BUILTIN };
#define CL_MAX_GROUPS 4
typedef struct cl_modset {
    uint64_t mask;                  /* universe bits present in the tuple        */
    uint8_t first[CL_MAX_GROUPS];   /* per mod_var choice group: universe bit of
                                       the first member in tuple order, or 0xFF
                                       (_match_opcode, patterns.py:163-166)      */
    uint16_t minus_wide;            /* modset id with WIDE removed (:416)        */
    uint16_t minus_x4;              /* modset id with X4 removed (frontend.py:542)*/
} cl_modset;
/* well-known modset ids (the encoder interns these first) */
enum { CL_MS_NONE = 0, CL_MS_LO, CL_MS_HI, CL_MS_S64, CL_MS_U64, CL_MS_F2I, CL_MS_I2F,
       CL_MS__WELLKNOWN };

/* value origin codes for values created on the device (ValueInfo.origin)     */
#define CL_ORG_HOST   0u            /* value existed on input; host keeps string  */
#define CL_ORG_PAIR   1u            /* "pair"             (patterns.py:292,356)  */
#define CL_ORG_BITS   (2u << 28)    /* origin(vid)+".bits" (:865)  | vid         */
#define CL_ORG_F      (3u << 28)    /* origin(vid)+".f"    (:874)  | vid         */
#define CL_ORG_KIND(o) ((o) >> 28 ? (o) >> 28 : (o))

typedef struct cl_corpus {       /* dense CSR at the ABI boundary              */
    uint32_t n_funcs, n_blocks, n_modsets, reserved;
    /* per function */
    cl_func *func;                  /* [n_funcs]                                */
    uint32_t *func_blk_off;         /* [n_funcs+1] block range of the function  */
    uint32_t *ext_off;              /* [n_funcs+1] overflow-slot region         */
    uint32_t *mem_off;              /* [n_funcs+1] memref region                */
    uint32_t *imm_off;              /* [n_funcs+1] immediate region             */
    uint32_t *val_off;              /* [n_funcs+1] value region (= next_vid each)*/
    /* per block */
    cl_blk *blk;                    /* [n_blocks], sorted by bid per function   */
    uint32_t *blk_off;              /* [n_blocks+1] instruction range           */
    /* instruction planes, [blk_off[n_blocks]] */
    cl_hdr *hdr;
    uint16_t *tag;                  /* [..][8]                                  */
    uint32_t *pay;                  /* [..][8]                                  */
    uint16_t *ext_tag;              /* [ext_off[n_funcs]]                       */
    uint32_t *ext_pay;
    cl_memref *mem;                 /* [mem_off[n_funcs]]                       */
    cl_imm *imm;                    /* [imm_off[n_funcs]]                       */
    /* value table, [val_off[n_funcs]] */
    uint8_t *val_alive;             /* vid in fn.values                         */
    int32_t *val_def_iid;           /* ValueInfo.def_iid, -1 = None             */
    uint32_t *val_origin;           /* CL_ORG_* (output only)                   */
    /* modifier-set table, [n_modsets] */
    const cl_modset *modsets;
} cl_corpus;

/* ---------------------------------------------------------- pattern table */
/* Compiled form of list[Pattern] (patterns.py:36-106, tables :531-664).      */
#define CL_MAX_PATTERNS 16
#define CL_MAX_TEMPLATES 3
#define CL_MAX_VARS 16
#define CL_PATTERN_MAGIC 0x434c5054u   /* "CLPT" */

enum cl_slot_kind { CL_S_ANY = 0, CL_S_VAR, CL_S_RZ, CL_S_PT, CL_S_IMM };
typedef struct cl_slot {
    uint8_t kind;       /* enum cl_slot_kind                                     */
    uint8_t var;        /* variable index (CL_S_VAR)                             */
    uint8_t neg;        /* 0 don't care, 1 must be False, 2 must be True         */
    uint8_t bitnot;     /* same encoding                                         */
    uint8_t half;       /* 0 don't care, 1 "H0", 2 "H1"                          */
    uint8_t pad[3];
    uint64_t imm;       /* LitImm.bits                                           */
} cl_slot;

typedef struct cl_template {    /* InstTemplate (patterns.py:67-75)              */
    uint16_t op;
    uint8_t n_defs, n_aux, n_uses, n_modvars;
    uint8_t modvar_var[2];      /* "mod:<var>" index, own namespace              */
    uint8_t modvar_group[2];    /* choice group id                               */
    uint8_t pad[6];
    uint64_t mods_all, mods_none;
    cl_slot slot[8];            /* defs, aux, uses                               */
} cl_template;

enum cl_rewrite {               /* the nine rewrites, patterns.py:324-511        */
    CL_RW_IADD364 = 0, CL_RW_ISETP64, CL_RW_LEA64, CL_RW_IMAD_WIDE, CL_RW_MOV64,
    CL_RW_CAST64, CL_RW_SHL64, CL_RW_SHR64, CL_RW_XMAD, CL_RW__COUNT
};

typedef struct cl_pattern {     /* Pattern (patterns.py:78-86)                   */
    uint8_t n_templates, rewrite, n_vars, table; /* table: 0 aggregation, 1 xmad */
    uint8_t var_a, var_b, var_c; /* CL_RW_XMAD: indices of $a $b $c             */
    uint8_t modvar_cond, modvar_bop; /* CL_RW_ISETP64: "mod:cond", "mod:bop"     */
    /* Join plan (host-derived from the slots, an optimisation only): every
     * template but the anchor defines a variable that an already resolved
     * template uses, so its instruction is the SSA definition of that operand
     * instead of a member of the candidate product (patterns.py:195).        */
    uint8_t join_ok;            /* 0: enumerate the product                       */
    uint8_t join_order[3];      /* templates in resolution order, [0] = anchor    */
    uint8_t join_from[3];       /* [k>=1]: resolved template holding the use      */
    uint8_t join_slot[3];       /* [k>=1]: its slot index (defs, aux, uses order) */
    uint8_t pad[13];
    cl_template t[CL_MAX_TEMPLATES];
} cl_pattern;

typedef struct cl_pattern_blob {
    uint32_t magic, n_patterns, n_groups, budget;  /* budget: 50_000 (:194)      */
    uint64_t group_mask[CL_MAX_GROUPS];   /* universe bits of each choice group   */
    uint8_t group_pos[64];                /* universe bit -> position in its group */
    uint16_t isetp64_ms[8][2][8];         /* [cond pos][U64][bop pos] -> modset id */
    cl_pattern p[CL_MAX_PATTERNS];
} cl_pattern_blob;

/* ------------------------------------------------------------ side outputs */
enum cl_event_kind {
    CL_EV_REFUSED = 1,   /* fn.diagnose("bb..: pattern .. refused") (patterns.py:684):
                            a = pattern index in the table of the phase, b = bid,
                            idx = rank of the match in select_matches order          */
    CL_EV_BOUNDARY = 2,  /* fn.meta["pattern_boundaries"] entry (:842): a = rcp vid,
                            b = add iid, idx = append order inside the function      */
    CL_EV_MATCH = 3      /* Match record (:100-106): a = pattern | selected << 16,
                            b, c, d = block positions of the matched instructions
                            (0xFFFFFFFF when the pattern is shorter); idx = pattern
                            << 20 | rank of the tuple in itertools.product order
                            (:195), which sorts like match_patterns' list, or
                            0x80000000 | rank in select_matches' list (:241)         */
};
/* seq = phase << 28 | index of the block inside its function; phase 0 = xmad
 * round, 1 = reciprocal (block index 0), 2.. = aggregation round 1...
 * cl_download() returns events sorted by (func, seq, kind, idx, a, b, c, d):
 * for REFUSED and BOUNDARY that is the reference's append order; for MATCH it
 * is the reference's product order (:187-203) within each block.              */
typedef struct cl_event {
    uint32_t func, seq, kind, idx, a, b, c, d;
} cl_event;

/* --------------------------------------------------------------- pass flags */
#define CL_PASS_XMAD       1u   /* normalize_xmad        patterns.py:805          */
#define CL_PASS_RECIPROCAL 2u   /* normalize_reciprocal  patterns.py:817          */
#define CL_PASS_AGGREGATE  4u   /* apply_aggregations    patterns.py:794          */
#define CL_PASS_TAG        8u   /* tag_cuda_objects      patterns.py:895          */
#define CL_PASS_ALL        15u
#define CL_PASS_MATCH_ONLY 16u  /* match_patterns + select_matches only (:181,:241):
                                   emit CL_EV_MATCH events, leave the stream alone  */
#define CL_PASS_MATCH_XMAD 32u  /* with MATCH_ONLY: use the xmad table            */

typedef struct cl_run_opts {
    uint32_t passes;        /* CL_PASS_*                                          */
    uint32_t max_rounds;    /* 4 (patterns.py:796)                                */
    uint32_t emit_matches;  /* also emit CL_EV_MATCH for every round of a full run */
    uint32_t reserved;
} cl_run_opts;

typedef struct cl_stats {
    uint64_t matches[CL_MAX_PATTERNS];    /* raw matches, all rounds              */
    uint64_t selected[CL_MAX_PATTERNS];   /* after select_matches                 */
    uint64_t rewrites[CL_MAX_PATTERNS];   /* successful rewrites                  */
    uint64_t refused[CL_MAX_PATTERNS];
    uint64_t n_inst_in, n_inst_out, n_events, reserved;
} cl_stats;

/* ------------------------------------------------------------------- C ABI */
typedef struct cl_ctx cl_ctx;

/* All functions return 0 on success, negative on error; cl_last_error()
 * describes the last failure on the calling thread.  A ctx is bound to one
 * device and is not thread safe; distinct ctxs are independent.              */
const char *cl_last_error(void);
const char *cl_backend(void);            /* "cuda-sm_100a" or "cpu-oracle"         */
/* sizeof() of the ABI structs as this library was compiled, for the binding's
 * layout check: 0 cl_hdr 1 cl_imm 2 cl_memref 3 cl_blk 4 cl_func 5 cl_modset
 * 6 cl_slot 7 cl_template 8 cl_pattern 9 cl_pattern_blob 10 cl_event
 * 11 cl_corpus 12 cl_run_opts 13 cl_stats 14 cl_sr_entry; -1 otherwise.      */
long cl_abi_sizeof(int which);
int cl_create(int device, cl_ctx **out);
void cl_destroy(cl_ctx *ctx);

/* PatternTable: replaces the module-level lists patterns.py:531/:634.        */
int cl_set_patterns(cl_ctx *ctx, const void *blob, size_t nbytes);

/* Host worker threads (oracle backend only; the CUDA backend ignores it).   */
int cl_set_threads(cl_ctx *ctx, int n_threads);

/* Copy a host corpus to the device (borrowed pointers, H2D inside).         */
int cl_upload(cl_ctx *ctx, const cl_corpus *in);

/* Post-SSA stage: replaces the call sequence pipeline.py:165-169
 * (normalize_xmad, normalize_reciprocal, apply_aggregations,
 * tag_cuda_objects) for every uploaded function.  Device resident; may be
 * called repeatedly on the same upload (it always restarts from the input).  */
int cl_run_postssa(cl_ctx *ctx, const cl_run_opts *opts);

/* Raw stage (functions uploaded as ONE block holding fn.raw_instructions):
 * CL_RAW_X4 replaces normalize_instruction (frontend.py:523-548: PT aux defs
 * dropped, .X4 -> explicit SHL feeding the address) on every instruction;
 * CL_RAW_SR replaces substitute_special_registers (frontend.py:697-722) with
 * `map` standing for arch.SR_CONST_OFFSETS (arch.py:33-39).  The register
 * group widening the reference runs between the two is host code outside the
 * path, so build_function (frontend.py:748-753) calls this twice.           */
#define CL_RAW_X4 1u
#define CL_RAW_SR 2u
typedef struct cl_sr_entry { uint32_t arch, offset, sreg; } cl_sr_entry; /* bank 0 */
int cl_run_raw(cl_ctx *ctx, uint32_t passes, const cl_sr_entry *map, uint32_t n_map);

/* Sizes of the result (dense), then the copy itself (D2H inside); `out`
 * arrays are caller allocated with the sizes reported in `sizes`:
 * func/blk tables keep their shape; sizes = {n_inst, n_ext, n_mem, n_imm,
 * n_val, n_events}.                                                          */
int cl_out_sizes(cl_ctx *ctx, uint64_t sizes[6]);
int cl_download(cl_ctx *ctx, cl_corpus *out, cl_event *events);

int cl_get_stats(cl_ctx *ctx, cl_stats *out);
/* Device time of the last cl_run_* in milliseconds (CUDA events on the
 * launching stream); the oracle reports host wall time.                      */
int cl_last_run_ms(cl_ctx *ctx, float *ms);
/* Device pointer of the per-pattern u64 match counters of the last run, for
 * the final ncclAllGather of the sharded driver (no host copy).  NULL on the
 * oracle backend.                                                            */
void *cl_device_counts_ptr(cl_ctx *ctx);
/* Stream used by the context (cudaStream_t as void*), NULL on the oracle.    */
void *cl_stream(cl_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CULIFTER_H */

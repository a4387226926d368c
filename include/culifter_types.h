/* culifter_types.h -- C ABI of the type-seeding step that follows the
 * normalisation + aggregation stage.
 *
 * Replaces typerec.seed_types (typerec.py:288-345) and the signature table it
 * consults, typerec.signature_for (typerec.py:78-235), for every function of
 * the corpus a context holds (cl_upload, culifter.h): one pass over the
 * instruction records that intersects ("narrows") the candidate type set of
 * every SSA value with what its defining and using instructions demand, and
 * records which instructions are type transparent (LINK constraints) for the
 * fixpoint that follows on the host (typerec.py:364-).
 *
 * Implemented by the same two libraries as culifter.h:
 *   paper_2604_27486_b200/csrc/libculifter.so  (product: sm_100a kernel)
 *   oracle/liboracle.so                        (TEST INFRASTRUCTURE)
 * Paths are relative to /root/reference/pkg/src/sasslift/.
 */
#ifndef CULIFTER_TYPES_H
#define CULIFTER_TYPES_H

#include "culifter.h"

#ifdef __cplusplus
extern "C" {
#endif

/* type lattice leaves as bits (lattice.py:13-23); a mask is a candidate set */
#define CL_TY_INT32   0x01u
#define CL_TY_FLOAT32 0x02u
#define CL_TY_INT64   0x04u
#define CL_TY_FLOAT64 0x08u
#define CL_TY_INT128  0x10u
#define CL_TY_BOOL    0x20u
#define CL_TY_FLOAT16 0x40u
#define CL_TY_BF16    0x80u
#define CL_TY_NUM32   (CL_TY_INT32 | CL_TY_FLOAT32)
#define CL_TY_NUM64   (CL_TY_INT64 | CL_TY_FLOAT64)
#define CL_TY_NUM128  CL_TY_INT128
#define CL_TY_TOP     0xFFu

/* which branch of signature_for (typerec.py:78-235) an opcode takes; derived
 * by the host from the base mnemonic and frontend.OPCODE_TABLE
 * (frontend.py:42-86) with the precedence of the reference's if-chain.       */
enum cl_sigkind {
    CL_SK_NONE = 0,   /* control, sync, opaque, unknown: no constraints (:234) */
    CL_SK_FALU, CL_SK_FSEL, CL_SK_FCMP, CL_SK_DALU, CL_SK_DCMP, CL_SK_HALU, CL_SK_HCMP,   /* :87-102 */
    CL_SK_IMAD,       /* IMAD/UIMAD: .WIDE form (:104) else plain ialu          */
    CL_SK_LOP, CL_SK_SHF, CL_SK_SHLR, CL_SK_IADD3, CL_SK_IADD, CL_SK_LEA,                 /* :109-126 */
    CL_SK_IALU, CL_SK_ICMP, CL_SK_PRED,                                                   /* :127-133 */
    CL_SK_MOV, CL_SK_SEL, CL_SK_SELECT, CL_SK_PHI, CL_SK_SREG, CL_SK_SHUFFLE, CL_SK_VOTE, /* :135-152 */
    CL_SK_I2F, CL_SK_F2I, CL_SK_F2F, CL_SK_I2I, CL_SK_FRND, CL_SK_CAST64, CL_SK_BITCAST,  /* :154-174 */
    CL_SK_LOAD, CL_SK_STORE, CL_SK_ATOMIC, CL_SK_TENSOR,                                  /* :176-214 */
    CL_SK_IADD364, CL_SK_ISETP64, CL_SK_LEA64, CL_SK_IMAD64, CL_SK_MOV64, CL_SK_SH64,
    CL_SK_PACK64, CL_SK_PACK128, CL_SK_UNPACK64, CL_SK_UNPACK128,                         /* :216-233 */
    CL_SK__COUNT
};
#define CL_OT_ADDR64 1u   /* MemRef uses are Int64: GLOBAL_SPACE loads/stores (:187,:196), ATOM/ATOMG (:205) */
#define CL_OT_RED    2u   /* RED: stored element follows the atomic rule (_store_elem, :238)  */
typedef struct cl_optype {        /* one per opcode id (fixed table + dynamic ids)    */
    uint8_t kind;                 /* enum cl_sigkind                                  */
    uint8_t flags;                /* CL_OT_*                                          */
} cl_optype;

#define CL_MT_WIDE 1u
#define CL_MT_HI   2u
#define CL_MT_F32  4u
#define CL_MT_F2I  8u
#define CL_MT_I2F  16u
typedef struct cl_modtype {       /* one per interned modifier tuple (cl_hdr.modset)  */
    uint8_t f16_elem;             /* _f16_elem  typerec.py:46                         */
    uint8_t mma_elem;             /* _mma_elem  :50                                   */
    uint8_t conv_float;           /* _conv_float(mods) :58                            */
    uint8_t conv_int;             /* _conv_int  :69                                   */
    uint8_t f2f_dst, f2f_src;     /* F2F: first / second float-format modifier (:158-162) */
    uint8_t atom_elem;            /* _atom_elem :243                                  */
    uint8_t flags;                /* CL_MT_*: "WIDE" "HI" "F32" "F2I" "I2F" in mods   */
} cl_modtype;

/* Host metadata the stream does not carry (Instruction.meta), as a sparse CSR keyed by the instruction id:
 * for function f the entries off[f] .. off[f+1]-1, sorted by iid.  Only loads, stores and tensor ops read it, and
 * the stage never rewrites those, so the same table serves the uploaded corpus and the stage's result.
 *   val bits 0..3   meta["packed_def_width"]  (0 = absent)            typerec.py:179
 *       bits 4..7   meta["packed_data_width"] (0 = absent, reads as 1) :191
 *       bits 8..15, 16..23, 24..31  meta["tensor_groups"] a, b, c     :209-210    */
typedef struct cl_typehints {
    const uint32_t *off;          /* [n functions + 1]                                */
    const uint32_t *iid;          /* [off[n functions]]                               */
    const uint32_t *val;
} cl_typehints;
#define CL_TH_DEFW(h)  ((h) & 15u)
#define CL_TH_DATAW(h) (((h) >> 4) & 15u)
#define CL_TH_NA(h)    (((h) >> 8) & 255u)
#define CL_TH_NB(h)    (((h) >> 16) & 255u)
#define CL_TH_NC(h)    ((h) >> 24)

/* which records are seeded */
#define CL_SEED_INPUT  0u   /* the corpus of the last cl_upload                                          */
#define CL_SEED_RESULT 1u   /* the dense result the last cl_run_postssa left on the device: the stage and the
                               seeding chain without a host round trip (pipeline.py:165-175); array sizes are
                               those of cl_out_sizes (records = sizes[0], values = sizes[4])              */

enum cl_role { CL_ROLE_SEED = 0, CL_ROLE_TRANSPARENT = 1, CL_ROLE_CONVERSION = 2 };
#define CL_LINK_ALL_FROM_15 0x8000u
#define CL_NO_VALUE 0xFFFFFFFFu

typedef struct cl_typeseed {      /* caller-allocated host arrays                     */
    uint32_t *val_masks;  /* [n values] TypeState.seed_mask | def_seed_mask << 8 | use_seed_mask << 16
                             (typerec.py:262-264), TOP where nothing narrowed         */
    uint8_t *role;        /* [n records] TypeState.roles[iid] (:311), enum cl_role    */
    uint16_t *link_mask;  /* [n records] bit k: use k (its ValueRef, or the ValueRef base of its MemRef)
                             is a member of link_uses (:326-329); bit 15 also stands for every use >= 15 */
    uint32_t *link_def;   /* [n records] vid of link_def (:316) or CL_NO_VALUE        */
    uint8_t *status;      /* [n functions] CL_ST_OK, or CL_ST_KEY_ERROR when a narrowed value is not in
                             fn.values (the reference's dict lookup raises KeyError, :301) */
} cl_typeseed;

/* seed_types over every function of the context's corpus (`source`), in one launch.
 * `ops[n_ops]` / `mods[n_mods]` cover every opcode id / modset id the corpus uses (ids beyond the tables are an
 * error); `hints` may be NULL (no instruction carries the three meta keys).  Device time of the call is reported
 * by cl_last_run_ms.                                                         */
int cl_seed_types(cl_ctx *ctx, uint32_t source, const cl_optype *ops, uint32_t n_ops,
                  const cl_modtype *mods, uint32_t n_mods,
                  const cl_typehints *hints, cl_typeseed *out);

#ifdef __cplusplus
}
#endif
#endif /* CULIFTER_TYPES_H */

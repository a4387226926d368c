/* kargs.h -- kernel parameter block and result directory shared by the
 * translation units of the CUDA library (culifter.cu, stream.cu). */
#pragma once
#include "core.cuh"

namespace clk { struct TileDesc { uint32_t first, nf; }; }      /* functions flist[first .. first + nf) */
using clk::TileDesc;
using clk::Caps;
using clk::PF__N;

/* ----------------------------------------------------------- kernel params */
struct FuncOut {               /* where a function's result lives (device)       */
    cl_func f;
    uint32_t inst_start, n_inst, imm_start, n_imm, val_start, ev_start, n_ev, pad;
};
enum { CUR_INST = 0, CUR_IMM, CUR_VAL, CUR_EV, CUR__N };

struct KArgs {
    cl_corpus in;              /* device pointers                               */
    const cl_pattern_blob *pb;
    const uint8_t *opflags;
    /* results: dense, in completion order; FuncOut says where                 */
    cl_hdr *o_hdr; uint16_t *o_tag; uint32_t *o_pay;
    cl_imm *o_imm;
    uint8_t *o_alive; int32_t *o_def_iid; uint32_t *o_origin;
    uint16_t *o_ext_tag; uint32_t *o_ext_pay; cl_memref *o_mem;      /* input offsets */
    cl_blk *o_blk; uint32_t *o_blk_start, *o_blk_cnt;                /* by global block */
    cl_event *o_ev;
    FuncOut *o_func;
    unsigned long long cap[CUR__N];
    unsigned long long *cursor;          /* [CUR__N]                            */
    unsigned long long *stats;           /* cl_stats as u64[]                   */
    unsigned long long *prof;            /* [PF__N] cycle counters               */
    /* work */
    const uint32_t *list; uint32_t n_list; uint32_t *work_counter;
    const uint32_t *n_list_ptr;          /* non-null: the list length lives on the device (retry list) */
    uint32_t *retry_list, *retry_count;  /* non-null: functions that outgrow this kernel's tight work
                                            memory are queued for the roomy one instead of failing   */
    uint8_t *scratch; unsigned long long scratch_per_group;
    Caps gcap;                 /* capacities of the scratch placement            */
    uint32_t hot_bytes;        /* shared memory per group for the hot arrays     */
    uint32_t passes, max_rounds, emit_matches, raw_passes;
    const cl_sr_entry *sr; uint32_t n_sr;
    /* tile kernel (tile.cuh) */
    const TileDesc *tiles; uint32_t n_tiles; uint32_t *tile_counter;
    const uint32_t *tile_flist;
    uint32_t *retry_big_list, *retry_big_count; uint32_t small_max;   /* hand-backs above small_max go to the CTA-group kernel */
    uint8_t *tile_scratch; unsigned long long tile_scratch_per_cta;   /* per group */
};


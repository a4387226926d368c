/* codec.c -- the host side of subsystem (1) of the north star, "pack the parsed
 * instruction stream once into struct-of-arrays": LiftedFunction objects ->
 * the planes of include/culifter.h, as a CPython extension.
 *
 * Same result, byte for byte, as soa.encode_py (the Python walk it replaces;
 * tests/test_codec.py compares the two on every golden fixture); about ten
 * times its speed, because the per-operand work is attribute reads and integer
 * packing.  What is read from the objects is what the reference's dataclasses
 * define: operands.py:41-255 (Opcode, Reg, UReg, Pred, ZeroReg, Imm, ConstMem,
 * SReg, MemRef, ValueRef), ssir.py:42-84 (Instruction), :189-235 (values),
 * :378-382 (terminator value uses).  The interned id tables (opcodes, modifier
 * tuples, strings) stay the Python objects of layout.TABLES: a hit is a dict
 * lookup, a miss calls the interning method.
 *
 * RAW-phase corpora (the two passes of the front half) keep the Python walk:
 * they are not on the headline path.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

enum { K_NONE, K_VALUE, K_IMM, K_RZ, K_URZ, K_PRED, K_REG, K_UREG, K_CONSTMEM, K_SREG, K_MEMREF };
enum { T_NEG = 1 << 4, T_NOT = 1 << 5, T_ABS = 1 << 6, T_HALF_SHIFT = 7, T_REUSE = 1 << 9, T_WIDTH_SHIFT = 10, T_IMM_FLOAT = 1 << 5 };
enum { CM_OFFSET_BITS = 20, SLOTS = 8, IF_EXT = 1, IF_GUARD = 2, IF_SYNTH = 4, IF_OBJ_SHIFT = 3, IF_OBJUSE_SHIFT = 5 };

typedef struct { uint8_t *p; size_t n, cap; } Buf;                  /* n, cap in bytes */
static int buf_room(Buf *b, size_t extra) {
    if (b->n + extra <= b->cap) return 0;
    size_t c = b->cap ? b->cap * 2 : 1 << 16;
    while (c < b->n + extra) c *= 2;
    uint8_t *q = (uint8_t *)PyMem_RawRealloc(b->p, c);
    if (!q) { PyErr_NoMemory(); return -1; }
    b->p = q; b->cap = c;
    return 0;
}
static int buf_put(Buf *b, const void *src, size_t n) {
    if (buf_room(b, n)) return -1;
    memcpy(b->p + b->n, src, n); b->n += n;
    return 0;
}
static PyObject *buf_bytes(Buf *b) { return PyBytes_FromStringAndSize((const char *)b->p, (Py_ssize_t)b->n); }

#pragma pack(push, 1)
typedef struct { uint32_t iid; uint16_t op, modset; uint8_t n_defs, n_aux, n_uses, flags; uint32_t ext; } Hdr;
typedef struct { uint64_t bits, text; } Imm;
typedef struct { uint16_t base_tag, ureg_tag; uint32_t base_pay, ureg_pay; int32_t off_hi; uint32_t off_lo; } MemRef;
typedef struct { uint32_t bid; uint16_t term_tag[2]; uint32_t term_pay[2]; } Blk;
typedef struct { uint32_t next_vid, next_iid, next_temp_reg; uint8_t arch, status; uint16_t reserved; } Func;
#pragma pack(pop)

/* interned attribute names */
static PyObject *s_vid, *s_negated, *s_absolute, *s_bitnot, *s_half, *s_bits, *s_text, *s_is_float, *s_uniform, *s_index,
    *s_base, *s_width, *s_reuse, *s_offset, *s_bank, *s_name, *s_ureg, *s_block_order, *s_bid, *s_instructions, *s_terminator,
    *s_cond, *s_guard, *s_meta, *s_cuda_object, *s_synthetic, *s_defs, *s_aux_defs, *s_uses, *s_iid, *s_opcode, *s_modifiers,
    *s_values, *s_def_iid, *s_next_vid, *s_next_iid, *s_next_temp_reg, *s_arch, *s_op_id, *s_modset_id, *s_str_id,
    *s_m_opcode, *s_m_modset, *s_m_string, *s_H0, *s_H1;

typedef struct {
    PyObject *tables, *op_id, *modset_id, *str_id, *err;      /* borrowed for the call */
    Buf hdr, tag, pay, ext_tag, ext_pay, mem, imm, blk, blk_cnt, func, alive, def_iid;
    Buf func_blk_off, ext_off, mem_off, imm_off, val_off;
    /* per function */
    size_t f_imm0, f_mem0, f_ext0;
    uint64_t *ik; uint32_t *iv; size_t icap, iused;             /* (bits, text) -> index, open addressing */
    /* operand type cache */
    PyTypeObject *tcache[16]; int tkind[16]; int ntc;
} Enc;

static PyObject *fail(Enc *e, const char *fmt, PyObject *obj) {
    PyObject *r = obj ? PyObject_Repr(obj) : NULL;
    PyErr_Format(e->err, fmt, r ? PyUnicode_AsUTF8(r) : "?");
    Py_XDECREF(r);
    return NULL;
}
/* getattr(o, name, False) as a truth value; -1 on error */
static int attr_true(PyObject *o, PyObject *name) {
    PyObject *v = PyObject_GetAttr(o, name);
    if (!v) { if (PyErr_ExceptionMatches(PyExc_AttributeError)) { PyErr_Clear(); return 0; } return -1; }
    const int t = PyObject_IsTrue(v);
    Py_DECREF(v);
    return t;
}
static int attr_ll(PyObject *o, PyObject *name, long long *out) {
    PyObject *v = PyObject_GetAttr(o, name);
    if (!v) return -1;
    *out = PyLong_AsLongLong(v);
    Py_DECREF(v);
    return (*out == -1 && PyErr_Occurred()) ? -1 : 0;
}
static int intern_id(Enc *e, PyObject *dict, PyObject *method, PyObject *key, long *out) {
    PyObject *v = PyDict_GetItemWithError(dict, key);              /* borrowed */
    if (v) { *out = PyLong_AsLong(v); return 0; }
    if (PyErr_Occurred()) return -1;
    v = PyObject_CallMethodObjArgs(e->tables, method, key, NULL);
    if (!v) return -1;
    *out = PyLong_AsLong(v);
    Py_DECREF(v);
    return 0;
}
static int flag_bits(PyObject *op, int absolute, int bitnot, unsigned *t) {
    int r = attr_true(op, s_negated); if (r < 0) return -1; if (r) *t |= T_NEG;
    if (bitnot) { r = attr_true(op, s_bitnot); if (r < 0) return -1; if (r) *t |= T_NOT; }
    if (absolute) { r = attr_true(op, s_absolute); if (r < 0) return -1; if (r) *t |= T_ABS; }
    return 0;
}
static int half_bits(Enc *e, PyObject *op, unsigned *t) {
    PyObject *h = PyObject_GetAttr(op, s_half);
    if (!h) { if (PyErr_ExceptionMatches(PyExc_AttributeError)) { PyErr_Clear(); return 0; } return -1; }
    int code = -1;
    if (h == Py_None) code = 0;
    else if (PyUnicode_Check(h)) {
        if (PyUnicode_Compare(h, s_H0) == 0) code = 1;
        else if (PyUnicode_Compare(h, s_H1) == 0) code = 2;
    }
    Py_DECREF(h);
    if (code < 0) { fail(e, "unsupported half selector on %s", op); return -1; }
    *t |= (unsigned)code << T_HALF_SHIFT;
    return 0;
}
static int kind_of_type(Enc *e, PyObject *op) {
    PyTypeObject *tp = Py_TYPE(op);
    for (int i = 0; i < e->ntc; i++) if (e->tcache[i] == tp) return e->tkind[i];
    static const struct { const char *n; int k; } names[] = {
        { "ValueRef", K_VALUE }, { "Imm", K_IMM }, { "ZeroReg", K_RZ }, { "Pred", K_PRED }, { "Reg", K_REG },
        { "UReg", K_UREG }, { "ConstMem", K_CONSTMEM }, { "SReg", K_SREG }, { "MemRef", K_MEMREF } };
    const char *nm = strrchr(tp->tp_name, '.');
    nm = nm ? nm + 1 : tp->tp_name;
    int k = -1;
    for (size_t i = 0; i < sizeof names / sizeof names[0]; i++) if (!strcmp(nm, names[i].n)) k = names[i].k;
    if (e->ntc < 16) { e->tcache[e->ntc] = tp; e->tkind[e->ntc] = k; e->ntc++; }
    return k;
}
static int imm_index(Enc *e, uint64_t bits, uint64_t text, uint32_t *idx) {
    if ((e->iused + 1) * 2 > e->icap) {
        const size_t nc = e->icap ? e->icap * 2 : 256;
        uint64_t *nk = (uint64_t *)PyMem_RawCalloc(nc * 2, sizeof(uint64_t));
        uint32_t *nv = (uint32_t *)PyMem_RawMalloc(nc * sizeof(uint32_t));
        if (!nk || !nv) { PyErr_NoMemory(); return -1; }
        memset(nv, 0xFF, nc * sizeof(uint32_t));
        for (size_t i = 0; i < e->icap; i++) if (e->iv[i] != 0xFFFFFFFFu) {
            size_t h = (size_t)((e->ik[2 * i] * 0x9E3779B97F4A7C15ull) ^ (e->ik[2 * i + 1] * 0xC2B2AE3D27D4EB4Full)) & (nc - 1);
            while (nv[h] != 0xFFFFFFFFu) h = (h + 1) & (nc - 1);
            nk[2 * h] = e->ik[2 * i]; nk[2 * h + 1] = e->ik[2 * i + 1]; nv[h] = e->iv[i];
        }
        PyMem_RawFree(e->ik); PyMem_RawFree(e->iv);
        e->ik = nk; e->iv = nv; e->icap = nc;
    }
    size_t h = (size_t)((bits * 0x9E3779B97F4A7C15ull) ^ (text * 0xC2B2AE3D27D4EB4Full)) & (e->icap - 1);
    while (e->iv[h] != 0xFFFFFFFFu) {
        if (e->ik[2 * h] == bits && e->ik[2 * h + 1] == text) { *idx = e->iv[h]; return 0; }
        h = (h + 1) & (e->icap - 1);
    }
    *idx = (uint32_t)((e->imm.n - e->f_imm0) / sizeof(Imm));
    e->ik[2 * h] = bits; e->ik[2 * h + 1] = text; e->iv[h] = *idx; e->iused++;
    Imm m = { bits, text };
    return buf_put(&e->imm, &m, sizeof m);
}

/* encode_operand of soa.py: -> tag, payload */
static int enc_operand(Enc *e, PyObject *op, unsigned *tag, uint32_t *pay) {
    const int kind = kind_of_type(e, op);
    unsigned t = 0;
    long long a, b, c;
    switch (kind) {
    case K_VALUE:
        if (flag_bits(op, 1, 1, &t) || half_bits(e, op, &t) || attr_ll(op, s_vid, &a)) return -1;
        *tag = K_VALUE | t; *pay = (uint32_t)a;
        return 0;
    case K_IMM: {
        PyObject *bits = PyObject_GetAttr(op, s_bits);
        if (!bits) return -1;
        const uint64_t ub = PyLong_AsUnsignedLongLongMask(bits);     /* op.bits & M64 */
        Py_DECREF(bits);
        if (ub == (uint64_t)-1 && PyErr_Occurred()) return -1;
        PyObject *text = PyObject_GetAttr(op, s_text);
        if (!text) return -1;
        long tid;
        const int r = intern_id(e, e->str_id, s_m_string, text, &tid);
        Py_DECREF(text);
        if (r) return -1;
        uint32_t idx;
        if (imm_index(e, ub, (uint64_t)tid, &idx)) return -1;
        int neg = attr_true(op, s_negated), fl = attr_true(op, s_is_float);
        if (neg < 0 || fl < 0) return -1;
        *tag = K_IMM | (neg ? T_NEG : 0) | (fl ? T_IMM_FLOAT : 0); *pay = idx;
        return 0;
    }
    case K_RZ: {
        const int u = attr_true(op, s_uniform);
        if (u < 0 || flag_bits(op, 0, 1, &t)) return -1;
        *tag = (u ? K_URZ : K_RZ) | t; *pay = 0;
        return 0;
    }
    case K_PRED: {
        const int neg = attr_true(op, s_negated);
        if (neg < 0 || attr_ll(op, s_index, &a)) return -1;
        *tag = K_PRED | (neg ? T_NEG : 0); *pay = (uint32_t)a;
        return 0;
    }
    case K_REG: {
        if (attr_ll(op, s_base, &a) || attr_ll(op, s_width, &b)) return -1;
        if (!(a >= 0 && a < 65536 && b > 0 && b < 65536)) { fail(e, "register out of range: %s", op); return -1; }
        const int ru = attr_true(op, s_reuse);
        if (ru < 0 || flag_bits(op, 1, 1, &t) || half_bits(e, op, &t)) return -1;
        *tag = K_REG | t | (ru ? T_REUSE : 0); *pay = (uint32_t)(a | b << 16);
        return 0;
    }
    case K_UREG:
        if (attr_ll(op, s_index, &a) || attr_ll(op, s_width, &b)) return -1;
        if (!(a >= 0 && a < 65536 && b > 0 && b < 65536)) { fail(e, "uniform register out of range: %s", op); return -1; }
        if (flag_bits(op, 1, 1, &t)) return -1;
        *tag = K_UREG | t; *pay = (uint32_t)(a | b << 16);
        return 0;
    case K_CONSTMEM:
        if (attr_ll(op, s_offset, &a) || attr_ll(op, s_bank, &b) || attr_ll(op, s_width, &c)) return -1;
        if (!(a >= 0 && a < (1 << CM_OFFSET_BITS) && b >= 0 && b < 4096 && c > 0 && c < 8)) { fail(e, "constant-memory operand out of range: %s", op); return -1; }
        if (flag_bits(op, 1, 0, &t) || half_bits(e, op, &t)) return -1;
        *tag = K_CONSTMEM | t | (unsigned)c << T_WIDTH_SHIFT; *pay = (uint32_t)(a | b << CM_OFFSET_BITS);
        return 0;
    case K_SREG: {
        PyObject *nm = PyObject_GetAttr(op, s_name);
        if (!nm) return -1;
        long sid;
        const int r = intern_id(e, e->str_id, s_m_string, nm, &sid);
        Py_DECREF(nm);
        if (r) return -1;
        *tag = K_SREG; *pay = (uint32_t)sid;
        return 0;
    }
    case K_MEMREF: {
        MemRef m; memset(&m, 0, sizeof m);
        PyObject *parts[2];
        parts[0] = PyObject_GetAttr(op, s_base);
        if (!parts[0]) return -1;
        parts[1] = PyObject_GetAttr(op, s_ureg);
        if (!parts[1]) { Py_DECREF(parts[0]); return -1; }
        unsigned tg[2] = { K_NONE, K_NONE }; uint32_t py[2] = { 0, 0 };
        int bad = 0;
        for (int k = 0; k < 2 && !bad; k++) if (parts[k] != Py_None) bad = enc_operand(e, parts[k], &tg[k], &py[k]);
        Py_DECREF(parts[0]); Py_DECREF(parts[1]);
        if (bad) return -1;
        PyObject *off = PyObject_GetAttr(op, s_offset);
        if (!off) return -1;
        PyObject *offi = PyNumber_Long(off);                       /* int(op.offset) */
        Py_DECREF(off);
        if (!offi) return -1;
        int ovf = 0;
        const long long o = PyLong_AsLongLongAndOverflow(offi, &ovf);
        Py_DECREF(offi);
        if (ovf) { fail(e, "address offset out of range: %s", op); return -1; }
        if (o == -1 && PyErr_Occurred()) return -1;
        m.base_tag = (uint16_t)tg[0]; m.ureg_tag = (uint16_t)tg[1]; m.base_pay = py[0]; m.ureg_pay = py[1];
        m.off_hi = (int32_t)(o >> 32); m.off_lo = (uint32_t)((uint64_t)o & 0xFFFFFFFFu);
        *tag = K_MEMREF; *pay = (uint32_t)((e->mem.n - e->f_mem0) / sizeof(MemRef));
        return buf_put(&e->mem, &m, sizeof m);
    }
    default:
        PyErr_Format(e->err, "cannot encode operand of type %s", Py_TYPE(op)->tp_name);
        return -1;
    }
}

static int put_u32(Buf *b, uint32_t v) { return buf_put(b, &v, 4); }

static int enc_inst(Enc *e, PyObject *fn, PyObject *inst) {
    unsigned tg[SLOTS]; uint32_t py[SLOTS];
    Hdr h; memset(&h, 0, sizeof h);
    unsigned flags = 0;
    PyObject *meta = PyObject_GetAttr(inst, s_meta);
    if (!meta) return -1;
    if (meta != Py_None && PyDict_Check(meta) && PyDict_GET_SIZE(meta)) {
        PyObject *obj = PyDict_GetItemWithError(meta, s_cuda_object);      /* borrowed */
        if (obj && PyObject_IsTrue(obj) == 1) {
            PyObject *k0 = PySequence_GetItem(obj, 0);
            if (!k0) { Py_DECREF(meta); return -1; }
            const char *ks = PyUnicode_Check(k0) ? PyUnicode_AsUTF8(k0) : "";
            int kind = !strcmp(ks, "block_sync") ? 1 : !strcmp(ks, "warp_group") ? 2 : !strcmp(ks, "collective") ? 3 : 0;
            Py_DECREF(k0);
            if (!kind) { Py_DECREF(meta); PyErr_SetString(PyExc_KeyError, "cuda_object kind"); return -1; }
            flags |= (unsigned)kind << IF_OBJ_SHIFT | 7u << IF_OBJUSE_SHIFT;
        } else if (PyErr_Occurred()) { Py_DECREF(meta); return -1; }
        PyObject *syn = PyDict_GetItemWithError(meta, s_synthetic);
        if (syn && PyObject_IsTrue(syn) == 1) {
            long long iid;
            if (attr_ll(inst, s_iid, &iid)) { Py_DECREF(meta); return -1; }
            flags |= IF_SYNTH; h.ext = (uint32_t)iid;          /* SSA phase: no donor table (soa.encode_py, raw only) */
        } else if (PyErr_Occurred()) { Py_DECREF(meta); return -1; }
    }
    Py_DECREF(meta);
    /* slots: [guard] defs aux uses */
    PyObject *groups[4];
    groups[0] = PyObject_GetAttr(inst, s_guard);
    if (!groups[0]) return -1;
    groups[1] = PyObject_GetAttr(inst, s_defs);
    groups[2] = groups[1] ? PyObject_GetAttr(inst, s_aux_defs) : NULL;
    groups[3] = groups[2] ? PyObject_GetAttr(inst, s_uses) : NULL;
    int rc = -1;
    size_t total = 0;
    Buf wide_t = { 0 }, wide_p = { 0 };
    if (!groups[3]) goto done;
    Py_ssize_t len[4] = { groups[0] != Py_None, 0, 0, 0 };
    for (int g = 1; g < 4; g++) {
        len[g] = PySequence_Size(groups[g]);
        if (len[g] < 0) goto done;
        if (len[g] > 255) { PyErr_Format(e->err, "an instruction has %zd operands in one group", len[g]); goto done; }
    }
    if (len[0]) flags |= IF_GUARD;
    total = (size_t)(len[0] + len[1] + len[2] + len[3]);
    {
        size_t k = 0;
        for (int g = 0; g < 4; g++) {
            for (Py_ssize_t j = 0; j < len[g]; j++) {
                PyObject *op = g == 0 ? groups[0] : PySequence_GetItem(groups[g], j);
                if (!op) goto done;
                unsigned t; uint32_t p;
                const int r = enc_operand(e, op, &t, &p);
                if (g) Py_DECREF(op);
                if (r) goto done;
                if (total <= SLOTS) { tg[k] = t; py[k] = p; }
                else { const uint16_t t16 = (uint16_t)t; if (buf_put(&wide_t, &t16, 2) || buf_put(&wide_p, &p, 4)) goto done; }
                k++;
            }
        }
    }
    if (total > SLOTS) {
        flags |= IF_EXT;
        h.ext = (uint32_t)((e->ext_tag.n - e->f_ext0) / 2);
        if (buf_put(&e->ext_tag, wide_t.p, wide_t.n) || buf_put(&e->ext_pay, wide_p.p, wide_p.n)) goto done;
        total = 0;
    }
    for (size_t k = total; k < SLOTS; k++) { tg[k] = K_NONE; py[k] = 0; }
    {
        long long iid;
        if (attr_ll(inst, s_iid, &iid)) goto done;
        PyObject *opc = PyObject_GetAttr(inst, s_opcode);
        if (!opc) goto done;
        PyObject *base = PyObject_GetAttr(opc, s_base), *mods = base ? PyObject_GetAttr(opc, s_modifiers) : NULL;
        Py_DECREF(opc);
        long oid = 0, mid = 0;
        int r = !mods;
        if (!r) r = intern_id(e, e->op_id, s_m_opcode, base, &oid);
        if (!r) {
            PyObject *key = PyTuple_Check(mods) ? (Py_INCREF(mods), mods) : PySequence_Tuple(mods);
            r = !key || intern_id(e, e->modset_id, s_m_modset, key, &mid);
            Py_XDECREF(key);
        }
        Py_XDECREF(base); Py_XDECREF(mods);
        if (r) goto done;
        h.iid = (uint32_t)iid; h.op = (uint16_t)oid; h.modset = (uint16_t)mid;
        h.n_defs = (uint8_t)len[1]; h.n_aux = (uint8_t)len[2]; h.n_uses = (uint8_t)len[3]; h.flags = (uint8_t)flags;
    }
    {
        uint16_t t16[SLOTS];
        for (int k = 0; k < SLOTS; k++) t16[k] = (uint16_t)tg[k];
        if (buf_put(&e->hdr, &h, sizeof h) || buf_put(&e->tag, t16, sizeof t16) || buf_put(&e->pay, py, sizeof py)) goto done;
    }
    rc = 0;
done:
    for (int g = 0; g < 4; g++) Py_XDECREF(groups[g]);
    PyMem_RawFree(wide_t.p); PyMem_RawFree(wide_p.p);
    (void)fn;
    return rc;
}

static int enc_function(Enc *e, PyObject *fn, PyObject *archs) {
    e->f_imm0 = e->imm.n; e->f_mem0 = e->mem.n; e->f_ext0 = e->ext_tag.n;
    if (e->icap) { memset(e->iv, 0xFF, e->icap * sizeof(uint32_t)); e->iused = 0; }
    PyObject *blocks = PyObject_CallMethodNoArgs(fn, s_block_order);
    if (!blocks) return -1;
    PyObject *it = PyObject_GetIter(blocks);
    Py_DECREF(blocks);
    if (!it) return -1;
    PyObject *b;
    int rc = 0;
    while (!rc && (b = PyIter_Next(it))) {
        Blk bk; memset(&bk, 0, sizeof bk);
        long long bid;
        PyObject *insts = NULL, *term = NULL;
        rc = attr_ll(b, s_bid, &bid);
        if (!rc) { insts = PyObject_GetAttr(b, s_instructions); term = insts ? PyObject_GetAttr(b, s_terminator) : NULL; rc = !term; }
        if (!rc) {
            bk.bid = (uint32_t)bid;
            if (term != Py_None) {
                const char *tn = strrchr(Py_TYPE(term)->tp_name, '.');
                tn = tn ? tn + 1 : Py_TYPE(term)->tp_name;
                const int is_condbr = !strcmp(tn, "CondBr");
                PyObject *names[2] = { s_cond, s_guard };
                for (int k = 0; k < 2 && !rc; k++) {
                    PyObject *ref = PyObject_GetAttr(term, names[k]);
                    if (!ref) { if (PyErr_ExceptionMatches(PyExc_AttributeError)) { PyErr_Clear(); continue; } rc = -1; break; }
                    if (ref != Py_None && !(k == 1 && !is_condbr)) {
                        unsigned t; uint32_t p;
                        rc = enc_operand(e, ref, &t, &p);
                        bk.term_tag[k] = (uint16_t)t; bk.term_pay[k] = p;
                    }
                    Py_DECREF(ref);
                }
            }
        }
        if (!rc) rc = buf_put(&e->blk, &bk, sizeof bk);
        if (!rc) {
            PyObject *seq = PySequence_Fast(insts, "block.instructions is not a sequence");
            if (!seq) rc = -1;
            else {
                const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
                rc = put_u32(&e->blk_cnt, (uint32_t)n);
                for (Py_ssize_t i = 0; i < n && !rc; i++) rc = enc_inst(e, fn, PySequence_Fast_GET_ITEM(seq, i));
                Py_DECREF(seq);
            }
        }
        Py_XDECREF(insts); Py_XDECREF(term); Py_DECREF(b);
    }
    Py_DECREF(it);
    if (rc || PyErr_Occurred()) return -1;
    /* value table (ssir.py:189-235) */
    long long nv, niid, ntemp = 1000;
    if (attr_ll(fn, s_next_vid, &nv) || attr_ll(fn, s_next_iid, &niid)) return -1;
    const size_t a0 = e->alive.n, d0 = e->def_iid.n;
    if (buf_room(&e->alive, (size_t)nv) || buf_room(&e->def_iid, (size_t)nv * 4)) return -1;
    memset(e->alive.p + a0, 0, (size_t)nv); e->alive.n += (size_t)nv;
    memset(e->def_iid.p + d0, 0xFF, (size_t)nv * 4); e->def_iid.n += (size_t)nv * 4;
    PyObject *values = PyObject_GetAttr(fn, s_values);
    if (!values) return -1;
    {
        PyObject *k, *v; Py_ssize_t pos = 0;
        if (!PyDict_Check(values)) { Py_DECREF(values); PyErr_SetString(PyExc_TypeError, "fn.values is not a dict"); return -1; }
        while (PyDict_Next(values, &pos, &k, &v)) {
            const long long vid = PyLong_AsLongLong(k);
            if (vid < 0 || vid >= nv) { Py_DECREF(values); if (!PyErr_Occurred()) PyErr_SetString(PyExc_IndexError, "value id outside [0, _next_vid)"); return -1; }
            e->alive.p[a0 + (size_t)vid] = 1;
            PyObject *di = PyObject_GetAttr(v, s_def_iid);
            if (!di) { Py_DECREF(values); return -1; }
            if (di != Py_None) { const int32_t x = (int32_t)PyLong_AsLong(di); memcpy(e->def_iid.p + d0 + (size_t)vid * 4, &x, 4); }
            Py_DECREF(di);
        }
    }
    Py_DECREF(values);
    PyObject *meta = PyObject_GetAttr(fn, s_meta);
    if (!meta) return -1;
    if (PyDict_Check(meta)) { PyObject *t = PyDict_GetItemWithError(meta, s_next_temp_reg); if (t) ntemp = PyLong_AsLongLong(t); }
    Py_DECREF(meta);
    if (PyErr_Occurred()) return -1;
    PyObject *arch = PyObject_GetAttr(fn, s_arch);
    if (!arch) return -1;
    const Py_ssize_t ai = PySequence_Index(archs, arch);
    Py_DECREF(arch);
    if (ai < 0) return -1;
    Func fr = { (uint32_t)nv, (uint32_t)niid, (uint32_t)ntemp, (uint8_t)ai, 0, 0 };
    if (buf_put(&e->func, &fr, sizeof fr)) return -1;
    if (put_u32(&e->func_blk_off, (uint32_t)(e->blk.n / sizeof(Blk))) || put_u32(&e->ext_off, (uint32_t)(e->ext_tag.n / 2)) ||
        put_u32(&e->mem_off, (uint32_t)(e->mem.n / sizeof(MemRef))) || put_u32(&e->imm_off, (uint32_t)(e->imm.n / sizeof(Imm))) ||
        put_u32(&e->val_off, (uint32_t)e->alive.n)) return -1;
    return 0;
}

/* encode(functions, tables, archs, error_class) -> dict of bytes */
static PyObject *py_encode(PyObject *self, PyObject *args) {
    PyObject *functions, *tables, *archs, *err;
    if (!PyArg_ParseTuple(args, "OOOO", &functions, &tables, &archs, &err)) return NULL;
    Enc e; memset(&e, 0, sizeof e);
    e.tables = tables; e.err = err;
    e.op_id = PyObject_GetAttr(tables, s_op_id);
    e.modset_id = e.op_id ? PyObject_GetAttr(tables, s_modset_id) : NULL;
    e.str_id = e.modset_id ? PyObject_GetAttr(tables, s_str_id) : NULL;
    PyObject *out = NULL, *seq = NULL;
    if (!e.str_id) goto done;
    seq = PySequence_Fast(functions, "functions is not a sequence");
    if (!seq) goto done;
    if (put_u32(&e.func_blk_off, 0) || put_u32(&e.ext_off, 0) || put_u32(&e.mem_off, 0) || put_u32(&e.imm_off, 0) || put_u32(&e.val_off, 0)) goto done;
    for (Py_ssize_t f = 0; f < PySequence_Fast_GET_SIZE(seq); f++)
        if (enc_function(&e, PySequence_Fast_GET_ITEM(seq, f), archs)) goto done;
    {
        static const char *names[] = { "hdr", "tag", "pay", "ext_tag", "ext_pay", "mem", "imm", "blk", "blk_cnt", "func", "val_alive",
                                       "val_def_iid", "func_blk_off", "ext_off", "mem_off", "imm_off", "val_off" };
        Buf *bufs[] = { &e.hdr, &e.tag, &e.pay, &e.ext_tag, &e.ext_pay, &e.mem, &e.imm, &e.blk, &e.blk_cnt, &e.func, &e.alive,
                        &e.def_iid, &e.func_blk_off, &e.ext_off, &e.mem_off, &e.imm_off, &e.val_off };
        out = PyDict_New();
        for (size_t i = 0; out && i < sizeof bufs / sizeof bufs[0]; i++) {
            PyObject *b = buf_bytes(bufs[i]);
            if (!b || PyDict_SetItemString(out, names[i], b)) { Py_XDECREF(b); Py_CLEAR(out); break; }
            Py_DECREF(b);
        }
    }
done:
    Py_XDECREF(seq); Py_XDECREF(e.op_id); Py_XDECREF(e.modset_id); Py_XDECREF(e.str_id);
    {
        Buf *bufs[] = { &e.hdr, &e.tag, &e.pay, &e.ext_tag, &e.ext_pay, &e.mem, &e.imm, &e.blk, &e.blk_cnt, &e.func, &e.alive,
                        &e.def_iid, &e.func_blk_off, &e.ext_off, &e.mem_off, &e.imm_off, &e.val_off };
        for (size_t i = 0; i < sizeof bufs / sizeof bufs[0]; i++) PyMem_RawFree(bufs[i]->p);
    }
    PyMem_RawFree(e.ik); PyMem_RawFree(e.iv);
    (void)self;
    return out;
}

static PyMethodDef methods[] = {
    { "encode", py_encode, METH_VARARGS, "encode(functions, tables, archs, error_class) -> {plane name: bytes}" },
    { NULL, NULL, 0, NULL } };
static struct PyModuleDef moddef = { PyModuleDef_HEAD_INIT, "_codec", "SoA encoder of culifter-b200 (see soa.py)", -1, methods };

PyMODINIT_FUNC PyInit__codec(void) {
#define S(v, text) if (!(v = PyUnicode_InternFromString(text))) return NULL
    S(s_vid, "vid"); S(s_negated, "negated"); S(s_absolute, "absolute"); S(s_bitnot, "bitnot"); S(s_half, "half"); S(s_bits, "bits");
    S(s_text, "text"); S(s_is_float, "is_float"); S(s_uniform, "uniform"); S(s_index, "index"); S(s_base, "base"); S(s_width, "width");
    S(s_reuse, "reuse"); S(s_offset, "offset"); S(s_bank, "bank"); S(s_name, "name"); S(s_ureg, "ureg"); S(s_block_order, "block_order");
    S(s_bid, "bid"); S(s_instructions, "instructions"); S(s_terminator, "terminator"); S(s_cond, "cond"); S(s_guard, "guard");
    S(s_meta, "meta"); S(s_cuda_object, "cuda_object"); S(s_synthetic, "synthetic"); S(s_defs, "defs"); S(s_aux_defs, "aux_defs");
    S(s_uses, "uses"); S(s_iid, "iid"); S(s_opcode, "opcode"); S(s_modifiers, "modifiers"); S(s_values, "values"); S(s_def_iid, "def_iid");
    S(s_next_vid, "_next_vid"); S(s_next_iid, "_next_iid"); S(s_next_temp_reg, "next_temp_reg"); S(s_arch, "arch"); S(s_op_id, "op_id");
    S(s_modset_id, "modset_id"); S(s_str_id, "str_id"); S(s_m_opcode, "opcode"); S(s_m_modset, "modset"); S(s_m_string, "string");
    S(s_H0, "H0"); S(s_H1, "H1");
#undef S
    return PyModule_Create(&moddef);
}

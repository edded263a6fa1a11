/*
 * TEST INFRASTRUCTURE -- the CPU oracle.  A plain-C restatement of the
 * reference's md_hom executor, used only by tests/, smoke() and bench.py's
 * cpu_baseline leg as the CHECKER.  The product path never links or calls it.
 *
 * Restates, step for step:
 *   - the stack-bytecode scalar VM        proj/src/engine.cpp:17-81 (compile_node)
 *                                          proj/src/engine.cpp:134-176 (Executor::leaf)
 *   - the strided accumulator + fold      proj/src/engine.cpp:92-112 (FoldOp),
 *                                          :177-189 (first-visit assign / fold), :313-335
 *   - the recursive loop nest             proj/src/engine.cpp:192-210 (step/walk),
 *                                          :215-220 (lex_plan); interpreter.cpp:54-66 (plan_from)
 *   - the prefix pass                     proj/src/engine.cpp:337-353
 *   - the output-view scatter             proj/src/views.cpp:242-275 (apply_output_view)
 *   - the test input generator            proj/tests/support.hpp:32-51 (make_inputs) over
 *                                          proj/include/mdh/rng.hpp:12-24 (mt19937_64)
 * The Python side (oracle/mdh_oracle.py) parses the spec and lowers it to the
 * flat tables these functions take, restating scalar_expr.cpp / views.cpp.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

/* ---- scalar VM (engine.cpp:17-21 Op enum, same instruction set) -------- */
enum {
  OP_LIT_I, OP_LIT_F, OP_IN_I, OP_IN_F, OP_IDX,
  OP_ADD_I, OP_ADD_F, OP_SUB_I, OP_SUB_F, OP_MUL_I, OP_MUL_F, OP_DIV_I, OP_DIV_F,
  OP_MIN_I, OP_MIN_F, OP_MAX_I, OP_MAX_F, OP_ABS_I, OP_ABS_F, OP_CMP_I, OP_CMP_F, OP_SELECT
};

typedef struct {
  int32_t op;
  int32_t arg;
  int64_t ilit;
  double flit;
} oracle_instr;

typedef union {
  int64_t i;
  double f;
} slot_t;

/* fold kinds: mda.hpp:52 BinOpKind {Add, Sub, Mul, Div, Min, Max} */
enum { FOLD_ADD = 0, FOLD_SUB = 1, FOLD_MUL = 2, FOLD_DIV = 3, FOLD_MIN = 4, FOLD_MAX = 5 };

static void fold_i(int kind, int64_t* acc, int64_t v) {
  switch (kind) {
    case FOLD_ADD: *acc += v; break;
    case FOLD_MUL: *acc *= v; break;
    case FOLD_MIN: *acc = v < *acc ? v : *acc; break;
    case FOLD_MAX: *acc = v > *acc ? v : *acc; break;
    default: break;
  }
}

static void fold_f(int kind, double* acc, double v) {
  switch (kind) {
    case FOLD_ADD: *acc += v; break;
    case FOLD_MUL: *acc *= v; break;
    case FOLD_MIN: *acc = v < *acc ? v : *acc; break;
    case FOLD_MAX: *acc = v > *acc ? v : *acc; break;
    default: break;
  }
}

typedef struct {
  int D;
  /* accesses in (buffer, access) flat order: engine.cpp:266-286 AccessPlan */
  int n_acc;
  const void* const* acc_data; /* base pointer of the buffer each access reads */
  const int64_t* acc_c0;
  const int64_t* acc_cj; /* [n_acc][D] */
  int64_t* acc_off;      /* current flat offset per access */
  /* programs: one per output component */
  int n_prog;
  const int32_t* prog_start;
  const int32_t* prog_len;
  const oracle_instr* code;
  const int32_t* prog_float;
  slot_t* stack;
  /* accumulator: engine.cpp:313-335 */
  const int64_t* acc_stride; /* [D], 0 on point-wise dims */
  int64_t acc_pos;
  void* const* acc_vals; /* per program: int64_t* or double* over acc cells */
  uint8_t* acc_def;
  int fold_kind;
  /* plan */
  int n_loops;
  const int32_t* loop_dim; /* 0-based */
  const int64_t* loop_count;
  const int64_t* loop_stride;
  int64_t* idx;
  int error;
  char* err;
  int errcap;
} exec_t;

static void set_err(exec_t* x, const char* msg) {
  if (!x->error) {
    x->error = 1;
    snprintf(x->err, (size_t)x->errcap, "%s", msg);
  }
}

static void leaf(exec_t* x) {
  for (int c = 0; c < x->n_prog; ++c) {
    const oracle_instr* code = x->code + x->prog_start[c];
    int len = x->prog_len[c];
    slot_t* st = x->stack;
    int sp = 0;
    for (int k = 0; k < len; ++k) {
      const oracle_instr* ins = &code[k];
      switch (ins->op) {
        case OP_LIT_I: st[sp++].i = ins->ilit; break;
        case OP_LIT_F: st[sp++].f = ins->flit; break;
        case OP_IN_I: st[sp++].i = ((const int64_t*)x->acc_data[ins->arg])[x->acc_off[ins->arg]]; break;
        case OP_IN_F: st[sp++].f = ((const double*)x->acc_data[ins->arg])[x->acc_off[ins->arg]]; break;
        case OP_IDX: st[sp++].i = x->idx[ins->arg]; break;
        case OP_ADD_I: --sp; st[sp - 1].i += st[sp].i; break;
        case OP_ADD_F: --sp; st[sp - 1].f += st[sp].f; break;
        case OP_SUB_I: --sp; st[sp - 1].i -= st[sp].i; break;
        case OP_SUB_F: --sp; st[sp - 1].f -= st[sp].f; break;
        case OP_MUL_I: --sp; st[sp - 1].i *= st[sp].i; break;
        case OP_MUL_F: --sp; st[sp - 1].f *= st[sp].f; break;
        case OP_DIV_I:
          --sp;
          if (st[sp].i == 0) {
            set_err(x, "DivisionByZero: integer division by zero in scalar function");
            return;
          }
          st[sp - 1].i /= st[sp].i;
          break;
        case OP_DIV_F: --sp; st[sp - 1].f /= st[sp].f; break;
        /* std::min(a, b) returns a unless b < a; std::max(a, b) returns a unless
           a < b (engine.cpp:166-169) -- matters for -0.0 / NaN */
        case OP_MIN_I: --sp; st[sp - 1].i = st[sp].i < st[sp - 1].i ? st[sp].i : st[sp - 1].i; break;
        case OP_MIN_F: --sp; st[sp - 1].f = st[sp].f < st[sp - 1].f ? st[sp].f : st[sp - 1].f; break;
        case OP_MAX_I: --sp; st[sp - 1].i = st[sp - 1].i < st[sp].i ? st[sp].i : st[sp - 1].i; break;
        case OP_MAX_F: --sp; st[sp - 1].f = st[sp - 1].f < st[sp].f ? st[sp].f : st[sp - 1].f; break;
        case OP_ABS_I: st[sp - 1].i = st[sp - 1].i < 0 ? -st[sp - 1].i : st[sp - 1].i; break;
        case OP_ABS_F: st[sp - 1].f = fabs(st[sp - 1].f); break;
        case OP_CMP_I:
          --sp;
          st[sp - 1].i = st[sp - 1].i < st[sp].i ? -1 : (st[sp - 1].i > st[sp].i ? 1 : 0);
          break;
        case OP_CMP_F:
          --sp;
          st[sp - 1].i = st[sp - 1].f < st[sp].f ? -1 : (st[sp - 1].f > st[sp].f ? 1 : 0);
          break;
        case OP_SELECT:
          sp -= 2;
          st[sp - 1] = st[sp - 1].i != 0 ? st[sp] : st[sp + 1];
          break;
        default: set_err(x, "Internal: bad opcode"); return;
      }
    }
    if (x->acc_def[x->acc_pos]) {
      if (x->prog_float[c])
        fold_f(x->fold_kind, &((double*)x->acc_vals[c])[x->acc_pos], st[0].f);
      else
        fold_i(x->fold_kind, &((int64_t*)x->acc_vals[c])[x->acc_pos], st[0].i);
    } else {
      if (x->prog_float[c])
        ((double*)x->acc_vals[c])[x->acc_pos] = st[0].f;
      else
        ((int64_t*)x->acc_vals[c])[x->acc_pos] = st[0].i;
    }
  }
  x->acc_def[x->acc_pos] = 1;
}

static void step(exec_t* x, int d, int64_t delta) {
  x->idx[d] += delta;
  x->acc_pos += x->acc_stride[d] * delta;
  for (int a = 0; a < x->n_acc; ++a) x->acc_off[a] += x->acc_cj[(size_t)a * (size_t)x->D + (size_t)d] * delta;
}

static void walk(exec_t* x, int lvl) {
  if (x->error) return;
  if (lvl == x->n_loops) {
    leaf(x);
    return;
  }
  int d = x->loop_dim[lvl];
  int64_t count = x->loop_count[lvl], stride = x->loop_stride[lvl];
  for (int64_t p = 0;;) {
    walk(x, lvl + 1);
    if (x->error) return;
    if (++p == count) break;
    step(x, d, stride);
  }
  step(x, d, -(count - 1) * stride);
}

/*
 * Runs the nest and leaves the folded accumulator (one array per output
 * component, acc_def marks visited cells).  Returns 0 or 1 (error in err).
 */
int oracle_run(int D, int n_acc, const void* const* acc_data, const int64_t* acc_c0, const int64_t* acc_cj,
               int n_prog, const int32_t* prog_start, const int32_t* prog_len, const oracle_instr* code,
               const int32_t* prog_float, int max_depth, const int64_t* acc_stride, void* const* acc_vals,
               uint8_t* acc_def, int fold_kind, int n_loops, const int32_t* loop_dim, const int64_t* loop_count,
               const int64_t* loop_stride, char* err, int errcap) {
  int64_t offs[256];
  int64_t idx[64];
  slot_t stack[512];
  if (n_acc > 256 || D > 64 || max_depth > 512) {
    snprintf(err, (size_t)errcap, "Unsupported: oracle limits exceeded");
    return 1;
  }
  exec_t x;
  memset(&x, 0, sizeof x);
  x.D = D;
  x.n_acc = n_acc;
  x.acc_data = acc_data;
  x.acc_c0 = acc_c0;
  x.acc_cj = acc_cj;
  x.acc_off = offs;
  for (int a = 0; a < n_acc; ++a) offs[a] = acc_c0[a];
  x.n_prog = n_prog;
  x.prog_start = prog_start;
  x.prog_len = prog_len;
  x.code = code;
  x.prog_float = prog_float;
  x.stack = stack;
  x.acc_stride = acc_stride;
  x.acc_vals = acc_vals;
  x.acc_def = acc_def;
  x.fold_kind = fold_kind;
  x.n_loops = n_loops;
  x.loop_dim = loop_dim;
  x.loop_count = loop_count;
  x.loop_stride = loop_stride;
  memset(idx, 0, sizeof idx);
  x.idx = idx;
  x.err = err;
  x.errcap = errcap;
  walk(&x, 0);
  return x.error;
}

/* Prefix pass over one ps dimension (engine.cpp:337-353). */
void oracle_prefix(int64_t acc_cells, int64_t stride, int64_t extent, int n_prog, const int32_t* prog_float,
                   void* const* acc_vals, const uint8_t* acc_def, int fold_kind) {
  for (int64_t flat = 0; flat < acc_cells; ++flat) {
    int64_t coord = (flat / stride) % extent;
    if (coord == 0) continue;
    if (!acc_def[flat] || !acc_def[flat - stride]) continue;
    for (int c = 0; c < n_prog; ++c) {
      if (prog_float[c])
        fold_f(fold_kind, &((double*)acc_vals[c])[flat], ((double*)acc_vals[c])[flat - stride]);
      else
        fold_i(fold_kind, &((int64_t*)acc_vals[c])[flat], ((int64_t*)acc_vals[c])[flat - stride]);
    }
  }
}

/*
 * Output-view scatter (views.cpp:242-275): every result cell r (lex order over
 * the collapsed ranges `coll`) is written through each output access; the
 * flat offset of access a is oc0[a] + sum_d ocj[a][d] * r_d.  Non-injective
 * writes must agree exactly.  comp_of_access[a] is the result component.
 */
int oracle_scatter(int D, const int64_t* coll, const int64_t* acc_stride, int n_oacc, const int64_t* oc0,
                   const int64_t* ocj, const int32_t* comp_of_access, const int32_t* comp_float,
                   void* const* out_data, uint8_t* const* out_def, void* const* acc_vals, char* err, int errcap) {
  int64_t r[64];
  int64_t cells = 1;
  for (int d = 0; d < D; ++d) {
    r[d] = 0;
    cells *= coll[d];
  }
  for (int64_t n = 0; n < cells; ++n) {
    int64_t flat = 0;
    for (int d = 0; d < D; ++d) flat += acc_stride[d] * r[d];
    for (int a = 0; a < n_oacc; ++a) {
      int64_t off = oc0[a];
      for (int d = 0; d < D; ++d) off += ocj[(size_t)a * (size_t)D + (size_t)d] * r[d];
      int c = comp_of_access[a];
      uint8_t* def = out_def[a];
      if (comp_float[c]) {
        double v = ((const double*)acc_vals[c])[flat];
        double* o = (double*)out_data[a];
        if (def[off]) {
          if (o[off] != v) {
            snprintf(err, (size_t)errcap, "InconsistentNonInjectiveWrite: disagreeing values at one cell");
            return 1;
          }
        } else {
          o[off] = v;
          def[off] = 1;
        }
      } else {
        int64_t v = ((const int64_t*)acc_vals[c])[flat];
        int64_t* o = (int64_t*)out_data[a];
        if (def[off]) {
          if (o[off] != v) {
            snprintf(err, (size_t)errcap, "InconsistentNonInjectiveWrite: disagreeing values at one cell");
            return 1;
          }
        } else {
          o[off] = v;
          def[off] = 1;
        }
      }
    }
    for (int d = D - 1; d >= 0; --d) {
      if (++r[d] < coll[d]) break;
      r[d] = 0;
    }
  }
  return 0;
}

/* ---- mt19937_64 (the standard engine; rng.hpp:12-24) ------------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}

static uint64_t mt64_next(mt64_t* g) {
  static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ MAG[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[(int)(x & 1ULL)];
    }
    x = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ MAG[(int)(x & 1ULL)];
    g->mti = 0;
  }
  uint64_t y = g->mt[g->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/*
 * make_inputs (support.hpp:32-51): one generator seeded with
 * seed * 0x9e3779b97f4a7c15 + 1, drawing below(11) - 5 for every cell of every
 * buffer in order; the integer k goes to out[] (callers scale f64 by 0.25).
 */
void oracle_make_inputs(uint64_t seed, int n_bufs, const int64_t* counts, int64_t* const* out) {
  static mt64_t g;
  mt64_seed(&g, seed * 0x9e3779b97f4a7c15ULL + 1ULL);
  for (int b = 0; b < n_bufs; ++b)
    for (int64_t t = 0; t < counts[b]; ++t) out[b][t] = (int64_t)(mt64_next(&g) % 11ULL) - 5;
}

/* Raw mt19937_64 stream, for pinning the generator against known values. */
void oracle_mt64(uint64_t seed, int64_t n, uint64_t* out) {
  static mt64_t g;
  mt64_seed(&g, seed);
  for (int64_t t = 0; t < n; ++t) out[t] = mt64_next(&g);
}

/* CPU restatement of the collective data path — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library, and only as the checker / CPU baseline; the product path
 * (liblagom_coll.so) never links or calls it.
 *
 * PARITY UNPINNED BY THE REFERENCE: the reference has no data-path
 * collective at all — a collective is only a traffic factor in comm_time
 * (reference proj/src/commperf.cpp:115-116, collective_factors in
 * proj/include/lagom/commperf.hpp:62-65). This file therefore restates the
 * standard (NCCL-compatible) semantics of the four collectives:
 *   ALL_GATHER      recv_r[k*B + i] = send_k[i]
 *   ALL_TO_ALL      recv_r[q*B + i] = send_q[r*B + i]
 *   REDUCE_SCATTER  recv_r[i]       = op over q of send_q[r*B + i]
 *   ALL_REDUCE      recv_r[i]       = op over q of send_q[i]
 * and fixes the ORDER of every floating-point reduction to the one the
 * sm_100a kernels use (paper_2602_20656_b200/csrc/coll/device.cuh), so fp32,
 * bf16 and fp16 results are compared bit for bit, not within a tolerance:
 *   ring (RS and AR):  block k is reduced along k+1, k+2, ..., k:
 *                      acc = x_{k+1}; acc = op(x_{k+2}, acc); ...; acc = op(x_k, acc)
 *                      (AR blocks are ring_block() = ceil(N/n) rounded up to
 *                      whole 16-byte packs)
 *   tree (AR):         binary tree, parent (v-1)/2:
 *                      val(v) = op(op(x_v, val(2v+1)), val(2v+2))
 * bf16/fp16 values are widened to fp32, combined once, and rounded back to
 * nearest-even — one rounding per hop, exactly as on the device.
 *
 * Multi-threaded with OpenMP over elements (bench.py's cpu_baseline states
 * the thread count it used).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { AR = 0, AG = 1, RS = 2, A2A = 3 };
enum { RING = 0, TREE = 1 };
enum { F32 = 0, BF16 = 1, F16 = 2, I32 = 3 };
enum { SUM = 0, MAX = 1, MIN = 2 };

static int esize(int dtype) { return (dtype == BF16 || dtype == F16) ? 2 : 4; }

static float bf16_to_f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float f16_to_f(uint16_t h) {
  _Float16 x;
  memcpy(&x, &h, 2);
  return (float)x;
}
static uint16_t f_to_f16(float f) {
  _Float16 x = (_Float16)f; /* IEEE round-to-nearest-even */
  uint16_t h;
  memcpy(&h, &x, 2);
  return h;
}

static float fop(int op, float a, float b) {
  return op == SUM ? a + b : op == MAX ? fmaxf(a, b) : fminf(a, b);
}

/* acc <- op(x, acc) on one element of the given dtype. */
static void combine(int dtype, int op, void* acc, const void* x) {
  switch (dtype) {
    case F32: {
      float a, b;
      memcpy(&a, acc, 4);
      memcpy(&b, x, 4);
      a = fop(op, b, a);
      memcpy(acc, &a, 4);
      break;
    }
    case I32: {
      int32_t a, b;
      memcpy(&a, acc, 4);
      memcpy(&b, x, 4);
      int32_t r = op == SUM ? (int32_t)((uint32_t)a + (uint32_t)b) : op == MAX ? (a > b ? a : b) : (a < b ? a : b);
      memcpy(acc, &r, 4);
      break;
    }
    case BF16: {
      uint16_t a, b;
      memcpy(&a, acc, 2);
      memcpy(&b, x, 2);
      uint16_t r = f_to_bf16(fop(op, bf16_to_f(b), bf16_to_f(a)));
      memcpy(acc, &r, 2);
      break;
    }
    case F16: {
      uint16_t a, b;
      memcpy(&a, acc, 2);
      memcpy(&b, x, 2);
      uint16_t r = f_to_f16(fop(op, f16_to_f(b), f16_to_f(a)));
      memcpy(acc, &r, 2);
      break;
    }
  }
}

/* AllReduce ring block size in elements (device.cuh ring_block). */
long long lagom_oracle_ring_block(long long count, int nranks, int dtype) {
  const long long pack = 16 / esize(dtype);
  const long long per = (count + nranks - 1) / nranks;
  return (per + pack - 1) / pack * pack;
}

static void tree_value(int dtype, int op, int n, int v, const char* const* send, long long byte_off,
                       char* out) {
  const int e = esize(dtype);
  char acc[4];
  memcpy(acc, send[v] + byte_off, (size_t)e);
  for (int c = 2 * v + 1; c <= 2 * v + 2 && c < n; ++c) {
    char sub[4];
    tree_value(dtype, op, n, c, send, byte_off, sub);
    /* acc <- op(acc, sub): the device combines own first, child second; the
     * ops are commutative, so op(sub, acc) has the same bits. */
    combine(dtype, op, acc, sub);
  }
  memcpy(out, acc, (size_t)e);
}

/* Parallel bulk copy (OpenMP over 1 MiB pieces): AllGather / AllToAll
 * blocks, the AllReduce broadcast and every single-rank collective. */
static void pcopy(char* dst, const char* src, long long bytes) {
  const long long piece = 1 << 20, np = (bytes + piece - 1) / piece;
  long long p;
#pragma omp parallel for schedule(static)
  for (p = 0; p < np; ++p) {
    const long long off = p * piece, len = bytes - off < piece ? bytes - off : piece;
    memcpy(dst + off, src + off, (size_t)len);
  }
}

/* Ring reduction of a run of m elements starting at element offset `first`,
 * for block k: acc = x_{k+1}; acc = op(x_{k+h}, acc) for h = 2..n, with the
 * element type's arithmetic inlined (widen, combine once, round at every
 * hop — the same bits as combine()). */
#define RING_RUN(T, LOAD, STORE, OPEXPR)                                       \
  {                                                                            \
    const T* xs[8];                                                            \
    for (int h = 1; h <= n; ++h) xs[h - 1] = (const T*)send[(k + h) % n] + first; \
    T* o = (T*)out;                                                            \
    long long i;                                                               \
    _Pragma("omp parallel for schedule(static)")                               \
    for (i = 0; i < m; ++i) {                                                  \
      T accr = xs[0][i];                                                       \
      for (int h = 1; h < n; ++h) {                                            \
        const float b = LOAD(xs[h][i]);                                        \
        const float a = LOAD(accr);                                            \
        accr = STORE(OPEXPR);                                                  \
      }                                                                        \
      o[i] = accr;                                                             \
    }                                                                          \
  }
static float id_f(float x) { return x; }
static float bf_ld(uint16_t h) { return bf16_to_f(h); }
static float h_ld(uint16_t h) { return f16_to_f(h); }

static void ring_run(int dtype, int op, int n, int k, const char* const* send, long long first, long long m,
                     char* out) {
  switch (dtype) {
    case F32:
      if (op == SUM) RING_RUN(float, id_f, id_f, b + a)
      else if (op == MAX) RING_RUN(float, id_f, id_f, fmaxf(b, a))
      else RING_RUN(float, id_f, id_f, fminf(b, a))
      return;
    case BF16:
      if (op == SUM) RING_RUN(uint16_t, bf_ld, f_to_bf16, b + a)
      else if (op == MAX) RING_RUN(uint16_t, bf_ld, f_to_bf16, fmaxf(b, a))
      else RING_RUN(uint16_t, bf_ld, f_to_bf16, fminf(b, a))
      return;
    case F16:
      if (op == SUM) RING_RUN(uint16_t, h_ld, f_to_f16, b + a)
      else if (op == MAX) RING_RUN(uint16_t, h_ld, f_to_f16, fmaxf(b, a))
      else RING_RUN(uint16_t, h_ld, f_to_f16, fminf(b, a))
      return;
    case I32: {
      const int32_t* xs[8];
      for (int h = 1; h <= n; ++h) xs[h - 1] = (const int32_t*)send[(k + h) % n] + first;
      int32_t* o = (int32_t*)out;
      long long i;
#pragma omp parallel for schedule(static)
      for (i = 0; i < m; ++i) {
        int32_t acc = xs[0][i];
        for (int h = 1; h < n; ++h) {
          const int32_t b = xs[h][i];
          acc = op == SUM ? (int32_t)((uint32_t)acc + (uint32_t)b) : op == MAX ? (acc > b ? acc : b)
                                                                               : (acc < b ? acc : b);
        }
        o[i] = acc;
      }
      return;
    }
  }
}

/* Computes every rank's output. send[r] / recv[r] are host buffers sized per
 * the count semantics of include/lagom_coll.h. Returns 0, or -1 on bad args. */
int lagom_oracle_collective(int coll, int algo, int nranks, int dtype, int op, long long count,
                            const void* const* send_v, void* const* recv_v) {
  if (nranks < 1 || nranks > 8 || count < 0) return -1;
  const char* const* send = (const char* const*)send_v;
  char* const* recv = (char* const*)recv_v;
  const int n = nranks, e = esize(dtype);
  const long long B = count;
  long long i;
  if (n == 1) {  /* every collective of one rank is a copy of its block */
    pcopy(recv[0], send[0], B * e);
    return 0;
  }
  switch (coll) {
    case AG:
      for (int r = 0; r < n; ++r)
        for (int k = 0; k < n; ++k) pcopy(recv[r] + k * B * e, send[k], B * e);
      return 0;
    case A2A:
      for (int r = 0; r < n; ++r)
        for (int q = 0; q < n; ++q) pcopy(recv[r] + q * B * e, send[q] + r * B * e, B * e);
      return 0;
    case RS:
      for (int r = 0; r < n; ++r) ring_run(dtype, op, n, r, send, r * B, B, recv[r]);
      return 0;
    case AR: {
      if (algo == TREE) {
#pragma omp parallel for schedule(static)
        for (i = 0; i < B; ++i) tree_value(dtype, op, n, 0, send, i * e, recv[0] + i * e);
      } else {
        const long long blk = lagom_oracle_ring_block(B, n, dtype);
        for (int k = 0; (long long)k * blk < B; ++k) {
          const long long first = (long long)k * blk, m = B - first < blk ? B - first : blk;
          ring_run(dtype, op, n, k, send, first, m, recv[0] + first * e);
        }
      }
      for (int r = 1; r < n; ++r) pcopy(recv[r], recv[0], B * e);
      return 0;
    }
  }
  return -1;
}

int lagom_oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

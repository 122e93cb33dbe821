/*
 * tir_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE (see tir_oracle.h).
 *
 * Naive loops restating tir::run on the operator programs emitted by
 * oracle/ir_gen.py. Generalises the reference's own naive oracles
 * (oracle_matmul / oracle_conv2d / oracle_depthwise, tests/testing/workloads.h:188-260)
 * to batch, stride, padding, dilation, groups, 1-D/3-D and the transposed
 * (gather) form. Multi-threaded over independent output rows only: every
 * output element's reduction order is unchanged, so the result is identical
 * for any thread count.
 */
#include "tir_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static int64_t floordiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
static int64_t floormod64(int64_t a, int64_t b) { return a - floordiv64(a, b) * b; }

int tir_oracle_conv_out(const tir_b200_conv_desc* d, int64_t out[3]) {
  const int64_t in[3] = {d->in_d, d->in_h, d->in_w};
  const int64_t k[3] = {d->k_d, d->k_h, d->k_w};
  const int64_t s[3] = {d->s_d, d->s_h, d->s_w};
  const int64_t p[3] = {d->p_d, d->p_h, d->p_w};
  const int64_t dl[3] = {d->d_d, d->d_h, d->d_w};
  for (int i = 0; i < 3; ++i) {
    if (in[i] < 1 || k[i] < 1 || s[i] < 1 || p[i] < 0 || dl[i] < 1) return -1;
    if (d->transposed) {
      out[i] = (in[i] - 1) * s[i] - 2 * p[i] + dl[i] * (k[i] - 1) + 1;
    } else {
      int64_t span = in[i] + 2 * p[i] - dl[i] * (k[i] - 1) - 1;
      if (span < 0) return -1;
      out[i] = span / s[i] + 1;
    }
    if (out[i] < 1) return -1;
  }
  return 0;
}

/* ---------------- GMM ---------------- */

typedef struct {
  const float *A, *B;
  float* C;
  int64_t M, N, K, r0, r1;
  int acc;
} gmm_job;

static void* gmm_worker(void* arg) {
  gmm_job* j = (gmm_job*)arg;
  for (int64_t i = j->r0; i < j->r1; ++i) {
    for (int64_t n = 0; n < j->N; ++n) {
      float acc = j->acc ? j->C[i * j->N + n] : 0.0f;
      for (int64_t k = 0; k < j->K; ++k) {
        float prod = j->A[i * j->K + k] * j->B[k * j->N + n];
        acc = acc + prod;
      }
      j->C[i * j->N + n] = acc;
    }
  }
  return NULL;
}

static void run_rows(void* (*fn)(void*), void* jobs, size_t job_size, int64_t rows, int threads,
                     void (*set_range)(void*, int64_t, int64_t)) {
  if (threads < 1) threads = 1;
  if (threads > rows) threads = (int)(rows > 0 ? rows : 1);
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    int64_t r0 = rows * t / threads, r1 = rows * (t + 1) / threads;
    void* job = (char*)jobs + job_size * (size_t)t;
    set_range(job, r0, r1);
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, fn, (char*)jobs + job_size * t);
  fn(jobs);
  for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
  free(tids);
}

static void gmm_set_range(void* j, int64_t r0, int64_t r1) {
  ((gmm_job*)j)->r0 = r0;
  ((gmm_job*)j)->r1 = r1;
}

int tir_oracle_gmm(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                   int accumulate, int threads) {
  if (M < 0 || N < 0 || K < 0) return -1;
  if (threads < 1) threads = 1;
  gmm_job* jobs = (gmm_job*)calloc((size_t)threads, sizeof(gmm_job));
  for (int t = 0; t < threads; ++t) {
    gmm_job j = {A, B, C, M, N, K, 0, 0, accumulate};
    jobs[t] = j;
  }
  run_rows(gmm_worker, jobs, sizeof(gmm_job), M, threads, gmm_set_range);
  free(jobs);
  return 0;
}

/* ---------------- convolution family ---------------- */

typedef struct {
  const tir_b200_conv_desc* d;
  const float *X, *W;
  float* Y;
  int64_t out[3];
  int64_t r0, r1; /* rows over n*OD*OH */
  int acc;
} conv_job;

static void* conv_worker(void* arg) {
  conv_job* j = (conv_job*)arg;
  const tir_b200_conv_desc* d = j->d;
  const int64_t ID = d->in_d, IH = d->in_h, IW = d->in_w;
  const int64_t OD = j->out[0], OH = j->out[1], OW = j->out[2];
  const int64_t G = d->groups, CIg = d->ci / G, COg = d->co / G, CO = d->co, CI = d->ci;
  for (int64_t row = j->r0; row < j->r1; ++row) {
    const int64_t oh = row % OH, od = (row / OH) % OD, n = row / (OH * OD);
    for (int64_t ow = 0; ow < OW; ++ow) {
      float* y = j->Y + (((n * OD + od) * OH + oh) * OW + ow) * CO;
      for (int64_t co = 0; co < CO; ++co) {
        const int64_t g = co / COg;
        float acc = j->acc ? y[co] : 0.0f;
        for (int64_t rd = 0; rd < d->k_d; ++rd) {
          for (int64_t rh = 0; rh < d->k_h; ++rh) {
            for (int64_t rw = 0; rw < d->k_w; ++rw) {
              int64_t id, ih, iw;
              int inb;
              if (d->transposed) {
                int64_t td = od + d->p_d - rd * d->d_d, th = oh + d->p_h - rh * d->d_h,
                        tw = ow + d->p_w - rw * d->d_w;
                id = floordiv64(td, d->s_d);
                ih = floordiv64(th, d->s_h);
                iw = floordiv64(tw, d->s_w);
                inb = floormod64(td, d->s_d) == 0 && floormod64(th, d->s_h) == 0 &&
                      floormod64(tw, d->s_w) == 0 && id >= 0 && id < ID && ih >= 0 && ih < IH &&
                      iw >= 0 && iw < IW;
              } else {
                id = od * d->s_d - d->p_d + rd * d->d_d;
                ih = oh * d->s_h - d->p_h + rh * d->d_h;
                iw = ow * d->s_w - d->p_w + rw * d->d_w;
                inb = id >= 0 && id < ID && ih >= 0 && ih < IH && iw >= 0 && iw < IW;
              }
              const float* x = inb ? j->X + (((n * ID + id) * IH + ih) * IW + iw) * CI + g * CIg
                                   : NULL;
              const float* w = j->W + ((rd * d->k_h + rh) * d->k_w + rw) * CIg * CO + co;
              for (int64_t rc = 0; rc < CIg; ++rc) {
                float a = inb ? x[rc] : 0.0f; /* select(inb, f32(A[..]), 0.0) */
                float prod = a * w[rc * CO];
                acc = acc + prod;
              }
            }
          }
        }
        y[co] = acc;
      }
    }
  }
  return NULL;
}

static void conv_set_range(void* j, int64_t r0, int64_t r1) {
  ((conv_job*)j)->r0 = r0;
  ((conv_job*)j)->r1 = r1;
}

int tir_oracle_conv(const tir_b200_conv_desc* d, const float* X, const float* W, float* Y,
                    int accumulate, int threads) {
  int64_t out[3];
  if (tir_oracle_conv_out(d, out) != 0) return -1;
  if (d->n < 1 || d->groups < 1 || d->ci % d->groups || d->co % d->groups) return -1;
  if (threads < 1) threads = 1;
  conv_job* jobs = (conv_job*)calloc((size_t)threads, sizeof(conv_job));
  for (int t = 0; t < threads; ++t) {
    conv_job j;
    memset(&j, 0, sizeof j);
    j.d = d;
    j.X = X;
    j.W = W;
    j.Y = Y;
    memcpy(j.out, out, sizeof out);
    j.acc = accumulate;
    jobs[t] = j;
  }
  run_rows(conv_worker, jobs, sizeof(conv_job), d->n * out[0] * out[1], threads, conv_set_range);
  free(jobs);
  return 0;
}

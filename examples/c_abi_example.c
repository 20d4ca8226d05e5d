/* Plain-C use of libtba.so (no Python, no PyTorch): build the rows of a tiny batch on the
 * host, copy them to the device with the CUDA runtime, run the VarGrad TB head forward and
 * backward through the C ABI, and print the loss, the per-sequence log-probs and a checksum
 * of dlogits; then the same sequences' log-probs from hidden states through the LM-head-fused
 * forward, and the loss with its gradients w.r.t. the hidden states and the LM-head weight
 * from the one-call LM-head forward + backward. The test suite runs it and compares with the
 * fp64 oracle.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_example.c \
 *       -L paper_2503_18929_b200 -ltba -L /usr/local/cuda/lib64 -lcudart -o c_abi_example
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tba.h"

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 2;                                                               \
    }                                                                         \
  } while (0)
#define TB(x)                                                                 \
  do {                                                                        \
    int r_ = (x);                                                             \
    if (r_ != TBA_OK) {                                                       \
      fprintf(stderr, "%s at %s:%d\n", tba_status_string(r_), __FILE__, __LINE__); \
      return 3;                                                               \
    }                                                                         \
  } while (0)

int main(int argc, char** argv) {
  const int64_t B = 2, K = 3, N = B * K, T = 4, V = 257;
  const double beta = 0.5;
  float* h_logits = (float*)malloc(sizeof(float) * N * T * V);
  int64_t* h_tok = (int64_t*)malloc(sizeof(int64_t) * N * T);
  uint8_t* h_mask = (uint8_t*)malloc(N * T);
  double h_ref[6], h_rew[6];
  uint64_t st = 88172645463325252ull; /* xorshift64: deterministic inputs */
  for (int64_t i = 0; i < N * T * V; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    h_logits[i] = (float)((double)(st >> 11) / 9007199254740992.0 * 8.0 - 4.0);
  }
  for (int64_t i = 0; i < N * T; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    h_tok[i] = (int64_t)(st % (uint64_t)V);
    h_mask[i] = (uint8_t)(i % T < T - (i / T) % 2); /* ragged: odd sequences drop the last token */
  }
  for (int s = 0; s < N; ++s) {
    h_ref[s] = -20.0 + s;
    h_rew[s] = (double)(s % 2);
  }
  float *d_logits, *d_dlogits;
  int64_t* d_tok;
  uint8_t* d_mask;
  double *d_ref, *d_rew, *d_seq, *d_logz, *d_resid, *d_partial;
  int32_t *d_ntok, *d_status;
  void* d_ws;
  const size_t ws = tba_workspace_bytes(N, T);
  CK(cudaMalloc((void**)&d_logits, sizeof(float) * N * T * V));
  CK(cudaMalloc((void**)&d_dlogits, sizeof(float) * N * T * V));
  CK(cudaMalloc((void**)&d_tok, sizeof(int64_t) * N * T));
  CK(cudaMalloc((void**)&d_mask, N * T));
  CK(cudaMalloc((void**)&d_ref, sizeof(double) * N));
  CK(cudaMalloc((void**)&d_rew, sizeof(double) * N));
  CK(cudaMalloc((void**)&d_seq, sizeof(double) * N));
  CK(cudaMalloc((void**)&d_logz, sizeof(double) * B));
  CK(cudaMalloc((void**)&d_resid, sizeof(double) * N));
  CK(cudaMalloc((void**)&d_partial, sizeof(double) * 3));
  CK(cudaMalloc((void**)&d_ntok, sizeof(int32_t) * N));
  CK(cudaMalloc((void**)&d_status, sizeof(int32_t)));
  CK(cudaMalloc(&d_ws, ws));
  CK(cudaMemcpy(d_logits, h_logits, sizeof(float) * N * T * V, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tok, h_tok, sizeof(int64_t) * N * T, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_mask, h_mask, N * T, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ref, h_ref, sizeof(h_ref), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rew, h_rew, sizeof(h_rew), cudaMemcpyHostToDevice));
  CK(cudaMemset(d_status, 0, sizeof(int32_t)));

  tba_rows rows;
  memset(&rows, 0, sizeof(rows));
  rows.logits = d_logits;
  rows.dtype = TBA_FP32;
  rows.n_seq = N;
  rows.seq_len = T;
  rows.vocab = V;
  rows.row_stride = V;
  rows.tokens = d_tok;
  rows.mask = d_mask;

  /* host-side validation happens before any CUDA work */
  if (tba_vargrad_tb_loss_fwd(&rows, d_ref, d_rew, 0.0, (int32_t)K, (double)N, d_ws, d_seq, d_ntok, d_logz, d_resid,
                              d_partial, d_status, NULL) != TBA_ERR_INVALID_CONFIG)
    return 4;
  TB(tba_vargrad_tb_loss_fwd(&rows, d_ref, d_rew, beta, (int32_t)K, (double)N, d_ws, d_seq, d_ntok, d_logz, d_resid,
                             d_partial, d_status, NULL));
  TB(tba_vargrad_tb_loss_bwd(&rows, d_ws, d_resid, 2.0 / (double)N, NULL, d_dlogits, TBA_FP32, V, NULL));
  CK(cudaDeviceSynchronize());

  double partial[3], seq[6];
  int32_t ntok[6], status;
  float* h_d = (float*)malloc(sizeof(float) * N * T * V);
  CK(cudaMemcpy(partial, d_partial, sizeof(partial), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(seq, d_seq, sizeof(seq), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ntok, d_ntok, sizeof(ntok), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&status, d_status, sizeof(status), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_d, d_dlogits, sizeof(float) * N * T * V, cudaMemcpyDeviceToHost));
  double cs = 0.0, rowsum = 0.0;
  for (int64_t i = 0; i < N * T * V; ++i) cs += fabs((double)h_d[i]);
  for (int64_t v = 0; v < V; ++v) rowsum += h_d[v];
  printf("abi %d status %d loss %.12g n_seq %.0f n_groups %.0f\n", tba_abi_version(), status, partial[0], partial[1],
         partial[2]);
  for (int s = 0; s < N; ++s) printf("seq %d logp %.12g ntok %d\n", s, seq[s], ntok[s]);
  printf("dlogits_abs_sum %.9g row0_sum %.3g\n", cs, rowsum);
  if (argc > 1) { /* the whole fp32 dlogits tensor, for an element-wise check against the oracle */
    FILE* f = fopen(argv[1], "wb");
    if (!f || fwrite(h_d, sizeof(float), (size_t)(N * T * V), f) != (size_t)(N * T * V)) return 3;
    fclose(f);
  }

  /* The LM-head-fused forward: the same sequences' log-probs from bf16 hidden states [N*T, D]
   * and an LM-head weight [V, D] (entries k/4, k in -2..2: exact in bf16, every logit exact in
   * fp32), run on the tensor cores without writing the logits. */
  const int64_t D = 64;
  uint16_t* h_hid = (uint16_t*)malloc(sizeof(uint16_t) * N * T * D);
  uint16_t* h_w = (uint16_t*)malloc(sizeof(uint16_t) * V * D);
  for (int64_t i = 0; i < N * T * D + V * D; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    float f = (float)((int)(st % 5u) - 2) * 0.25f;
    uint32_t b;
    memcpy(&b, &f, sizeof(b));
    if (i < N * T * D) h_hid[i] = (uint16_t)(b >> 16);
    else h_w[i - N * T * D] = (uint16_t)(b >> 16);
  }
  void *d_hid, *d_w, *d_lws;
  const size_t lws = tba_lmhead_workspace_bytes(N, T, V);
  CK(cudaMalloc(&d_hid, sizeof(uint16_t) * N * T * D));
  CK(cudaMalloc(&d_w, sizeof(uint16_t) * V * D));
  CK(cudaMalloc(&d_lws, lws));
  CK(cudaMemcpy(d_hid, h_hid, sizeof(uint16_t) * N * T * D, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_w, h_w, sizeof(uint16_t) * V * D, cudaMemcpyHostToDevice));
  tba_lmhead lm;
  memset(&lm, 0, sizeof(lm));
  lm.hidden = d_hid;
  lm.weight = d_w;
  lm.n_seq = N;
  lm.seq_len = T;
  lm.d = D;
  lm.vocab = V;
  lm.hidden_stride = D;
  lm.weight_stride = D;
  lm.tokens = d_tok;
  lm.mask = d_mask;
  TB(tba_lmhead_seq_logprob(&lm, 1.0, d_lws, d_seq, d_ntok, d_status, NULL));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(seq, d_seq, sizeof(seq), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&status, d_status, sizeof(status), cudaMemcpyDeviceToHost));
  for (int s = 0; s < N; ++s) printf("lmhead seq %d logp %.12g\n", s, seq[s]);

  /* Training step through the LM head in one call: loss, dL/dhidden (fp32) and dL/dW (fp32),
   * the [N, T, V] logits never allocated. */
  void *d_bws, *d_dh, *d_dw;
  const size_t bws = tba_lmhead_fwd_bwd_workspace_bytes(N, T, D, V, (int32_t)K, 0);
  CK(cudaMalloc(&d_bws, bws));
  CK(cudaMalloc(&d_dh, sizeof(float) * N * T * D));
  CK(cudaMalloc(&d_dw, sizeof(float) * V * D));
  TB(tba_lmhead_tb_loss_fwd_bwd(&lm, NULL, d_ref, d_rew, beta, (int32_t)K, (double)N, 2.0 / (double)N, 0, d_lws,
                                d_seq, d_ntok, d_logz, d_resid, d_partial, d_dh, TBA_FP32, D, (float*)d_dw, D, 0,
                                NULL, d_bws, d_status, NULL));
  CK(cudaDeviceSynchronize());
  float* h_dh = (float*)malloc(sizeof(float) * N * T * D);
  float* h_dw = (float*)malloc(sizeof(float) * V * D);
  CK(cudaMemcpy(partial, d_partial, sizeof(partial), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_dh, d_dh, sizeof(float) * N * T * D, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_dw, d_dw, sizeof(float) * V * D, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&status, d_status, sizeof(status), cudaMemcpyDeviceToHost));
  double sh = 0.0, sw = 0.0;
  for (int64_t i = 0; i < N * T * D; ++i) sh += fabs((double)h_dh[i]);
  for (int64_t i = 0; i < V * D; ++i) sw += fabs((double)h_dw[i]);
  printf("lmhead loss %.12g dhidden_abs_sum %.9g dweight_abs_sum %.9g\n", partial[0], sh, sw);
  return status != 0;
}

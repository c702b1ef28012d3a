/*
 * A non-Python caller of the C-ABI (include/mcf.h): dlopen libmcf.so, build
 * the items layout with mcf_csr_build, plan it with mcf_als_plan and solve
 * one weighted-lambda items half-step with mcf_als_half_step -- the calls a
 * C/C++ host of the reference's als_half_step (factor.py:512-538) would make.
 * Test infrastructure (tests/test_gpu_abi.py compiles and runs it).
 *
 * usage: mcf_driver <libmcf.so> <in.bin> <out.bin>
 *   in.bin : int64 nnz, U, I, D; float lam; int32 users[nnz], items[nnz];
 *            float scores[nnz], P[U*D], Q[I*D]
 *   out.bin: int64 fail_row; float Q_new[I*D]
 */
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mcf.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 2; } } while (0)
#define SYM(name) __typeof__(&name) p_##name = (__typeof__(&name))dlsym(h, #name); \
    if (!p_##name) { fprintf(stderr, "missing symbol %s\n", #name); return 3; }

static void *dev_copy(const void *src, size_t n) {
    void *d = NULL;
    if (cudaMalloc(&d, n ? n : 1) != cudaSuccess) return NULL;
    if (n && cudaMemcpy(d, src, n, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
    return d;
}

int main(int argc, char **argv) {
    if (argc != 4) { fprintf(stderr, "usage: %s lib in out\n", argv[0]); return 1; }
    void *h = dlopen(argv[1], RTLD_NOW | RTLD_LOCAL);
    if (!h) { fprintf(stderr, "dlopen: %s\n", dlerror()); return 3; }
    SYM(mcf_last_error) SYM(mcf_factor_ld) SYM(mcf_csr_workspace_bytes) SYM(mcf_csr_build)
    SYM(mcf_als_plan_bytes) SYM(mcf_als_plan) SYM(mcf_als_workspace_bytes) SYM(mcf_als_half_step)

    FILE *f = fopen(argv[2], "rb");
    if (!f) return 4;
    int64_t hdr[4]; float lam;
    if (fread(hdr, 8, 4, f) != 4 || fread(&lam, 4, 1, f) != 1) return 4;
    const int64_t nnz = hdr[0], U = hdr[1], I = hdr[2], D = hdr[3];
    int32_t *users = malloc(4 * nnz), *items = malloc(4 * nnz);
    float *scores = malloc(4 * nnz), *P = malloc(4 * U * D), *Q = malloc(4 * I * D);
    if (fread(users, 4, nnz, f) != (size_t)nnz || fread(items, 4, nnz, f) != (size_t)nnz ||
        fread(scores, 4, nnz, f) != (size_t)nnz || fread(P, 4, U * D, f) != (size_t)(U * D) ||
        fread(Q, 4, I * D, f) != (size_t)(I * D)) return 4;
    fclose(f);

    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    const int ld = p_mcf_factor_ld((int)D);
    /* factor tables [rows][ld], zero padding */
    float *Pp = calloc(U * ld, 4), *Qp = calloc(I * ld, 4);
    for (int64_t r = 0; r < U; ++r) memcpy(Pp + r * ld, P + r * D, 4 * D);
    float *dP = dev_copy(Pp, 4 * U * ld), *dQ = NULL;
    CK(cudaMalloc((void **)&dQ, 4 * I * ld));
    CK(cudaMemset(dQ, 0, 4 * I * ld));
    int32_t *du = dev_copy(users, 4 * nnz), *di = dev_copy(items, 4 * nnz);
    float *ds = dev_copy(scores, 4 * nnz);
    if (!dP || !du || !di || !ds) return 2;

    /* items layout (CSC): rows keyed by item, partner = user */
    int64_t *ptr; int32_t *idx; float *val; void *ws;
    CK(cudaMalloc((void **)&ptr, 8 * (I + 1)));
    CK(cudaMalloc((void **)&idx, 4 * nnz));
    CK(cudaMalloc((void **)&val, 4 * nnz));
    size_t wsb = p_mcf_csr_workspace_bytes(nnz, (int32_t)I);
    CK(cudaMalloc(&ws, wsb));
    int rc = p_mcf_csr_build(di, du, ds, nnz, (int32_t)I, ptr, idx, val, NULL, ws, wsb, s);
    if (rc) { fprintf(stderr, "mcf_csr_build: %s\n", p_mcf_last_error()); return 5; }
    CK(cudaFree(ws));

    const int chunk = 2048;
    int64_t info[MCF_PLAN_INFO_LEN];
    void *plan;
    size_t pb = p_mcf_als_plan_bytes((int32_t)I, nnz, chunk);
    CK(cudaMalloc(&plan, pb));
    rc = p_mcf_als_plan(ptr, NULL, (int32_t)I, 0, chunk, nnz, plan, pb, info, s);
    if (rc) { fprintf(stderr, "mcf_als_plan: %s\n", p_mcf_last_error()); return 5; }
    const int64_t slots = D <= 20 ? info[3] : info[1];
    size_t hb = p_mcf_als_workspace_bytes((int32_t)I, slots, (int32_t)D);
    CK(cudaMalloc(&ws, hb ? hb : 256));
    int64_t *fail;
    CK(cudaMalloc((void **)&fail, 8));
    /* weighted lambda: lam_c = 0, lam_n = lam */
    rc = p_mcf_als_half_step(ptr, idx, val, NULL, dP, U, dQ, (int32_t)D, 0.f, lam, 0.f, NULL,
                             NULL, 0.f, NULL, (int32_t)I, 0, chunk, plan, info, fail, NULL, ws,
                             hb, s);
    if (rc) { fprintf(stderr, "mcf_als_half_step: %s\n", p_mcf_last_error()); return 5; }
    CK(cudaStreamSynchronize(s));
    int64_t fail_h;
    CK(cudaMemcpy(&fail_h, fail, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Qp, dQ, 4 * I * ld, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < I; ++r) memcpy(Q + r * D, Qp + r * ld, 4 * D);

    FILE *o = fopen(argv[3], "wb");
    if (!o) return 4;
    fwrite(&fail_h, 8, 1, o);
    fwrite(Q, 4, I * D, o);
    fclose(o);
    printf("ok fail_row=%lld\n", (long long)fail_h);
    return 0;
}

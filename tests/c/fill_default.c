/* A non-Python host of the C-ABI (what a cgo / JNI / plain-C caller does):
 * default tables from the library, one production fill, raw f64le out.
 *
 *   fill_default <dist 0..3> <n> <seed> <ctr_base> <out.bin>
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "zigfast_b200.h"

int main(int argc, char** argv) {
    if (argc != 6) {
        fprintf(stderr, "usage: %s dist n seed ctr_base out.bin\n", argv[0]);
        return 2;
    }
    const int dist = atoi(argv[1]);
    const uint64_t n = strtoull(argv[2], NULL, 10);
    const uint64_t seed = strtoull(argv[3], NULL, 10);
    const uint64_t base = strtoull(argv[4], NULL, 10);
    zf_tables* t = NULL;
    int rc = (dist == ZF_TRAD_EXP || dist == ZF_TRAD_NORMAL) ? zf_trad_tables_create_default(0, &t)
                                                              : zf_tables_create_default(0, &t);
    if (rc != ZF_OK) {
        fprintf(stderr, "tables: %s\n", zf_strerror(rc));
        return 1;
    }
    double* dev = NULL;
    if (cudaMalloc((void**)&dev, n * sizeof(double)) != cudaSuccess) return 1;
    rc = zf_fill(t, dist, ZF_F64, seed, base, dev, n, NULL, NULL);
    if (rc != ZF_OK) {
        fprintf(stderr, "fill: %s\n", zf_strerror(rc));
        return 1;
    }
    double* host = (double*)malloc(n * sizeof(double));
    if (cudaMemcpy(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    FILE* f = fopen(argv[5], "wb");
    if (!f || fwrite(host, sizeof(double), n, f) != n) return 1;
    fclose(f);
    free(host);
    cudaFree(dev);
    zf_tables_destroy(t);
    return 0;
}

// tc_advance.cuh -- tcgen05 recurrent update (placeholder until the kernel lands)
#pragma once
#include "common.cuh"
static int tc_advance_launch(const DevModel &m, int prec, uint32_t n_cap, const uint32_t *n_dev,
                             const int32_t *in_row, const int32_t *words, const float *h_base,
                             float *out_base, const uint32_t *out_row0, cudaStream_t s) {
    return -1;
}

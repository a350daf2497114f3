/*
 * softmax.h -- C4 row statistics with a fixed summation order, shared by
 * gen_host.c and gen_device.cu so both produce identical bytes.
 *
 * Row r of `cols` logits l_c = 4 z_c.  m = max_c l_c (order-free).
 * e_c = exp(l_c - m) in fp64.  S = sum over lanes L = 0..31 (in order) of
 * partial_L, where partial_L = sum over c = L, L+32, L+64, ... (in order).
 * p_c = (float)(e_c / S).
 */
#ifndef SCAN_INPUTS_SOFTMAX_H
#define SCAN_INPUTS_SOFTMAX_H
#include "recipe.h"

INPUTS_HD double inputs_softmax_lane_partial(uint64_t seed, uint64_t row, uint64_t cols,
                                             uint32_t lane, float m)
{
    double s = 0.0;
    for (uint64_t c = lane; c < cols; c += 32)
        s = s + inputs_exp((double)inputs_softmax_logit(seed, row, cols, c) - (double)m);
    return s;
}

INPUTS_HD float inputs_softmax_value(uint64_t seed, uint64_t row, uint64_t cols, uint64_t c,
                                     float m, double S)
{
    double e = inputs_exp((double)inputs_softmax_logit(seed, row, cols, c) - (double)m);
    return (float)(e / S);
}
#endif

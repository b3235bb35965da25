// fields.cuh -- K2/K3/K4 entry points.
#pragma once
#include "common.cuh"

int fold_currents(const b200pic_state &st, cudaStream_t s);
int sync_fields(const b200pic_state &st, int comp0, int ncomp, cudaStream_t s);
int maxwell(b200pic_state &st, cudaStream_t s);
int maxwell_lagged(const b200pic_state &st, cudaStream_t s);
int sync_axes(const b200pic_state &st, int comp0, int ncomp, int axis_mask, cudaStream_t s);
int fold_axes(const b200pic_state &st, int axis_mask, cudaStream_t s);
int yee_half_b(const b200pic_state &st, cudaStream_t s);
int yee_full_e(const b200pic_state &st, cudaStream_t s);
int yee_pin_walls(const b200pic_state &st, cudaStream_t s);
int maxwell_slab(const b200pic_state &st, cudaStream_t s);
size_t xplanes_bytes(const b200pic_config &c, int which);
int xplanes_pack(const b200pic_state &st, int which, void *to_left, void *to_right, cudaStream_t s);
int xplanes_unpack(const b200pic_state &st, int which, const void *from_left, const void *from_right, cudaStream_t s);

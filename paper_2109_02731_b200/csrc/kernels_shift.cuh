// kernels_shift.cuh -- Pack / VectorPack / Shift kernels.
#pragma once
#include "kernels_core.cuh"
struct fdfb_ctx;
struct fdfb_params;
static size_t shift_pack_bytes(const fdfb_params& p);
static int pack_keygen(const fdfb_ctx* c, u64 seed, const int8_t* s_rlwe, void* pack, u64* shat, u64* tmask,
                       u64* tprod, u64* tout, int CH, cudaStream_t st);
static int pack_import(const fdfb_ctx* c, const u64* canon, void* dev, cudaStream_t st);

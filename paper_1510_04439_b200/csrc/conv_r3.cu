// K3 instantiations, padded radius buckets 32 and 48 (see conv_impl.cuh, conv.cuh).
#include "conv_impl.cuh"

DFPCA_CONV_INSTANTIATE(32)
DFPCA_CONV_INSTANTIATE(48)

// The BK = 32 / 2-stage configuration of the DMMA GEMM (namespace bgp::bk32),
// used for 512 tiles; see gemm.cu.
#define BGP_GEMM_BK32
#define BGP_GEMM_NS bk32
#define BGP_GEMM_SECONDARY
#include "gemm.cu"

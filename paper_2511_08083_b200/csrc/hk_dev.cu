// Development builds (HK_DEBUG_HANG, HK_TRACE, A/B variants): the product ABI and the
// diagnostics in ONE library, so a trace reader sees the event table of the kernels it traced
// and an A/B script can launch single backward phases of the same build. Release builds use
// the two libraries (libhkattn.so, libhkattn_diag.so) instead.
#include "hk_attn.cu"
#include "hk_diag.cu"

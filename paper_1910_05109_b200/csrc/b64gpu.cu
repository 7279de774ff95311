// b64gpu.cu -- single translation unit of libb64gpu.so (whole-program
// compilation: the templated kernels are instantiated and launched in one TU).
#include "encode.cu"
#include "decode.cu"
#include "unaligned.cu"
#include "peer.cu"
#include "group.cu"
#include "small.cu"
#include "mime.cu"
#include "stream.cu"
#include "offsets.cu"
#include "batch.cu"
#include "capi.cu"
#include "capi_ext.cu"

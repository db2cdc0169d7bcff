// Unity translation unit for libmenndl_sm100.so: the kernels are header
// templates, so one TU keeps every kernel instantiated exactly once.
#include "net.cu"
#include "kernel_abi.cu"

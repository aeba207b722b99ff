// RT_K_POLICY — fused acting step (placeholder until the fused MLP policy
// kernel lands; the planner never emits it yet).
#include "common.cuh"
extern "C" void* rt_kernel_policy(const void* params) { (void)params; return nullptr; }

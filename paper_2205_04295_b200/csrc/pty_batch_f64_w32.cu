// explicit instantiation of the batched extension for double, W = 32
#include "pty_batched_host.cuh"
namespace pty {
template int run_batch_contrib<double, 32>(const PtyBatchArgs*, cudaStream_t);
template int run_batch_apply<double, 32>(const PtyBatchArgs*, cudaStream_t);
template int64_t batch_workspace<double, 32>(int, int, int, int, bool);
}

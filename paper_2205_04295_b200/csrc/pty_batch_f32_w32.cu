// explicit instantiation of the batched extension for float, W = 32
#include "pty_batched_host.cuh"
namespace pty {
template int run_batch_contrib<float, 32>(const PtyBatchArgs*, cudaStream_t);
template int run_batch_apply<float, 32>(const PtyBatchArgs*, cudaStream_t);
template int64_t batch_workspace<float, 32>(int, int, int, int, bool);
}

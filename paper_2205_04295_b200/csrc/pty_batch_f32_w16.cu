// explicit instantiation of the batched extension for float, W = 16
#include "pty_batched_host.cuh"
namespace pty {
template int run_batch_contrib<float, 16>(const PtyBatchArgs*, cudaStream_t);
template int run_batch_apply<float, 16>(const PtyBatchArgs*, cudaStream_t);
template int64_t batch_workspace<float, 16>(int, int, int, int, bool);
}

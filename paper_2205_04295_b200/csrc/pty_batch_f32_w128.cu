// explicit instantiation of the batched extension for float, W = 128
#include "pty_batched_host.cuh"
namespace pty {
template int run_batch_contrib<float, 128>(const PtyBatchArgs*, cudaStream_t);
template int run_batch_apply<float, 128>(const PtyBatchArgs*, cudaStream_t);
template int64_t batch_workspace<float, 128>(int, int, int, int, bool);
}

// explicit instantiation of the batched extension for double, W = 64
#include "pty_batched_host.cuh"
namespace pty {
template int run_batch_contrib<double, 64>(const PtyBatchArgs*, cudaStream_t);
template int run_batch_apply<double, 64>(const PtyBatchArgs*, cudaStream_t);
template int64_t batch_workspace<double, 64>(int, int, int, int, bool);
}

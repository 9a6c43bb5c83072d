// explicit instantiation of the batched extension for double, W = 512
#include "pty_batched_host.cuh"
namespace pty {
template int run_batch_contrib<double, 512>(const PtyBatchArgs*, cudaStream_t);
template int run_batch_apply<double, 512>(const PtyBatchArgs*, cudaStream_t);
template int64_t batch_workspace<double, 512>(int, int, int, int, bool);
}

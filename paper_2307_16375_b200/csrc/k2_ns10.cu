// K2 instantiations for NS = 10 strategies (split per NS for parallel compilation).
#include "chain_dp.cuh"
namespace uniap {
template k2_fn k2_get<10>(int, int, bool, bool, bool);
}

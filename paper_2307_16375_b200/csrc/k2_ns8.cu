// K2 instantiations for NS = 8 strategies (split per NS for parallel compilation).
#include "chain_dp.cuh"
namespace uniap {
template k2_fn k2_get<8>(int, int, bool, bool, bool);
}

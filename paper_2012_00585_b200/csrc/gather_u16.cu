// Instantiation unit: the numeric kernels for uint16_t row-relative positions (split from
// numeric.cu so the two position widths compile in parallel).
#include "kernels.cuh"

namespace feagpu {

void gather_u16(fea_plan* p, const Incidences& in, const double* K, double* values, bool accumulate,
               cudaStream_t s) {
    gather<uint16_t>(p, in, K, values, accumulate, s);
}

void scatter_u16(fea_plan* p, const double* K, const int32_t* list, int64_t n_list, double* values,
                bool atomic, cudaStream_t s) {
    if (atomic && list == p->order.as<int32_t>() && n_list == p->E && atomic_staged<uint16_t>(p, K, values, s)) return;
    if (atomic) scatter<uint16_t, true>(p, K, list, n_list, values, s);
    else scatter<uint16_t, false>(p, K, list, n_list, values, s);
}

}  // namespace feagpu

// md.cu -- molecular-dynamics cell-pair path (see below).
#include <cstring>

#include "common.cuh"

namespace gc {
void md_kernel_spec(const char *cls, int64_t out[5])
{
    (void)cls;
    throw Error{GC_E_VALUE, "md kernel class not built yet"};
}
}  // namespace gc

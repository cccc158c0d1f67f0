// Peer memory for the fused row-partitioned assembly + gather (include/fea_gpu.h, fea_ipc_*).
// The root's global values buffer is exported as a CUDA IPC handle; each rank maps it and the
// numeric kernels store its owned row block straight into it at the block's global offset, so
// the row-block gather travels over NVLink/NVSwitch while the block is being assembled (no
// separate collective after the kernel). Plain pointers cross the ABI; torch allocates.
#include <cuda.h>

#include <cstring>

#include "internal.cuh"

namespace feagpu {
extern thread_local std::string g_err;
}

using namespace feagpu;

namespace {
template <class F>
fea_status guarded_p(F&& f) {
    try {
        g_err.clear();
        f();
        return FEA_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FEA_ERR_INVALID;
    }
}

// cuMemGetAddressRange through the runtime's driver entry point (the library links cudart
// statically and does not link libcuda itself)
using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
GetRangeFn get_range_fn() {
    static GetRangeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<GetRangeFn>(f);
    }();
    return fn;
}
}  // namespace

extern "C" {

fea_status fea_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset_bytes) {
    return guarded_p([&] {
        FEA_REQUIRE(dev_ptr && handle64 && offset_bytes, FEA_ERR_INVALID, "bad arguments");
        GetRangeFn fn = get_range_fn();
        FEA_REQUIRE(fn, FEA_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
        CUdeviceptr base = 0;
        size_t size = 0;
        FEA_REQUIRE(fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) == CUDA_SUCCESS, FEA_ERR_INVALID,
                    "pointer is not a device allocation");
        cudaIpcMemHandle_t h;
        FEA_CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
        static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
        std::memcpy(handle64, &h, sizeof(h));
        *offset_bytes = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    });
}

fea_status fea_ipc_open(const void* handle64, int device, void** base) {
    return guarded_p([&] {
        FEA_REQUIRE(handle64 && base, FEA_ERR_INVALID, "bad arguments");
        DeviceScope ds(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        FEA_CK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

fea_status fea_ipc_close(void* base) {
    return guarded_p([&] {
        FEA_REQUIRE(base, FEA_ERR_INVALID, "base is NULL");
        FEA_CK(cudaIpcCloseMemHandle(base));
    });
}

}  // extern "C"

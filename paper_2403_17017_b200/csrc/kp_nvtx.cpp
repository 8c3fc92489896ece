// kp_nvtx.cpp -- NVTX ranges for the C-ABI entry points (domain "kernelpick").
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

namespace kp {

static nvtxDomainHandle_t domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("kernelpick");
    return d;
}

struct NvtxRange {
    explicit NvtxRange(const char *name);
    ~NvtxRange();
};

NvtxRange::NvtxRange(const char *name) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(domain(), &a);
}

NvtxRange::~NvtxRange() { nvtxDomainRangePop(domain()); }

// Table III order (kernelpick_b200.h KP_* indices)
const char *kernel_label(int32_t kernel) {
    static const char *names[] = {"Adaptive-CSR", "CSR,BM", "CSR,MP", "CSR,WM",
                                  "CSR,WO",       "CSR,TM", "COO,WM", "ELL,TM"};
    return kernel >= 0 && kernel < 8 ? names[kernel] : "?";
}

}  // namespace kp

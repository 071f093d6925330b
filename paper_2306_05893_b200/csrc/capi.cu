// Error reporting and launch accounting shared by every libtsb entry point.
#include <atomic>
#include <cstring>
#include <string>

#include "tsb_common.cuh"

namespace tsb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_last_error(const std::string &msg) { g_last_error = msg; }
void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace tsb

extern "C" int tsb_abi_version(void) { return TSB_ABI_VERSION; }

extern "C" int tsb_last_error(char *buf, size_t len) {
    if (buf == nullptr || len == 0) return TSB_E_ARG;
    const std::string &m = tsb::g_last_error;
    size_t k = m.size() < len - 1 ? m.size() : len - 1;
    std::memcpy(buf, m.data(), k);
    buf[k] = '\0';
    return TSB_OK;
}

extern "C" int64_t tsb_launch_count(void) { return tsb::g_launches.load(); }

extern "C" int64_t tsb_struct_size(int32_t which) {
    switch (which) {
        case 0: return sizeof(tsb_asm_plan);
        case 1: return sizeof(tsb_asm_coeffs);
        case 2: return sizeof(tsb_ldlt_block);
        case 3: return sizeof(tsb_ldlt_desc);
        case 4: return sizeof(tsb_report);
        case 5: return sizeof(tsb_ldlt_tile);
        case 6: return sizeof(tsb_front);
        case 7: return sizeof(tsb_front_pair);
        case 8: return sizeof(tsb_refactor_desc);
        case 9: return sizeof(tsb_pattern);
        default: return -1;
    }
}

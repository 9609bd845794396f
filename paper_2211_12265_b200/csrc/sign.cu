// sign.cu -- placeholder until the persistent signing kernel lands
#include "engine.cuh"
namespace dlb {
template <class P>
int sign_dev(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*, const uint64_t*,
             const uint8_t*, size_t, int, uint8_t*, uint32_t*, uint8_t*, dlb_sign_stats*) {
  return DLB_E_ARG;
}
template int sign_dev<Params<2>>(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*, const uint64_t*, const uint8_t*, size_t, int, uint8_t*, uint32_t*, uint8_t*, dlb_sign_stats*);
template int sign_dev<Params<3>>(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*, const uint64_t*, const uint8_t*, size_t, int, uint8_t*, uint32_t*, uint8_t*, dlb_sign_stats*);
template int sign_dev<Params<5>>(dlb_ctx*, size_t, const uint8_t*, size_t, const uint8_t*, const uint64_t*, const uint8_t*, size_t, int, uint8_t*, uint32_t*, uint8_t*, dlb_sign_stats*);
}
extern "C" int dlb_dbg_sign_attempt(dlb_ctx*, int, size_t, const uint8_t*, size_t, const uint8_t*, const uint8_t*, const uint32_t*, uint8_t*, uint8_t*, int32_t*, int32_t*) { return DLB_E_ARG; }

// tc_path.cu — bf16 tcgen05 step (placeholder until the fused kernel lands).
#include "common.cuh"
namespace lcae {
struct TcScratch {};
lcae_status tc_alloc(lcae_layer *) { set_error("bf16 tcgen05 path not built yet"); return LCAE_ERR_CONFIG; }
void tc_free(lcae_layer *L) { delete L->tc; L->tc = nullptr; }
lcae_status tc_step(lcae_layer *, bool, bool) { set_error("bf16 path not built"); return LCAE_ERR_CONFIG; }
}  // namespace lcae

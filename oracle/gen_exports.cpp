// gen_exports.cpp — the oracle library's handle on the shared seeded input
// generator (paper_2408_14947_b200/csrc/datagen.cpp, compiled into this
// library with hidden visibility so its erx_gen_* names never interpose on
// the product library's).  TEST INFRASTRUCTURE ONLY, like the rest of oracle/.
#include "../include/erx_datagen.h"

extern "C" {
__attribute__((visibility("default"))) int orc_gen_preset(int config_id, uint32_t stream, void* spec_out) {
    return erx_gen_preset(config_id, stream, static_cast<erx_gen_spec*>(spec_out));
}
__attribute__((visibility("default"))) int orc_gen_lines(const void* spec, uint32_t first_line, uint32_t n_lines,
                                                         float* out, uint8_t* mask, int threads) {
    return erx_gen_lines(static_cast<const erx_gen_spec*>(spec), first_line, n_lines, out, mask, threads);
}
__attribute__((visibility("default"))) int orc_gen_scene_changes(const void* spec, int64_t* out) {
    return erx_gen_scene_changes(static_cast<const erx_gen_spec*>(spec), out);
}
}

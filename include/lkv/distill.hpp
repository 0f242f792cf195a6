// lkv/distill.hpp -- only the task-generator configuration that the evictsim interface names
// (proj/include/lkv/distill.hpp:67-83).  Training (distillation) is outside this B200 build.
#pragma once

namespace lkv {

struct TaskGenConfig {
    int min_len = 64;
    int max_len = 256;
    int n_records = 4;
    int record_repeats = 2;
    int record_marker = 1;
    int query_marker = 2;
    int key_base = 16;
    int n_keys = 32;
    int value_base = 96;
    int n_values = 64;
    int filler_base = 226;
    int n_filler = 24;
};

}  // namespace lkv

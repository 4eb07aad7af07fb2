// Test infrastructure: the reference includes <nlohmann/json_fwd.hpp> from its
// git-ignored vendor/ tree (proj/CMakeLists.txt:5). The image ships the full
// nlohmann/json 3.11.3 single header (cudnn_frontend wheel); forward to it.
#pragma once
#include <nlohmann/json.hpp>

// errors.h -- the thread-local message behind brmq_last_error(), shared by the
// CUDA solver layer (api.cu) and the host-only harness (harness.cpp).
#pragma once

namespace brmq {
int set_error(int code, const char* msg);  // stores msg, returns code
}

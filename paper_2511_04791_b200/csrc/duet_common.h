// Shared host-side helpers of libduet.so: thread-local error state and status macros.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/duet.h"

namespace duet {

void set_error(const char* fmt, ...);
void clear_error();

}  // namespace duet

#define DUET_FAIL(code, ...)            \
  do {                                  \
    ::duet::set_error(__VA_ARGS__);     \
    return (code);                      \
  } while (0)

#define DUET_TRY(expr)                  \
  do {                                  \
    duet_status s_ = (expr);            \
    if (s_ != DUET_OK) return s_;       \
  } while (0)

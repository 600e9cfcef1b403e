// Shared host helpers for libfvb: thread-local last-error message.
#pragma once
#include <cstdarg>
#include <cstdio>

void fvb_set_error(const char* fmt, ...);

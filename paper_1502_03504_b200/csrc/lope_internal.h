// lope_internal.h — helpers shared by the translation units of liblope_b200.so.
#pragma once

// Sets lope_last_error() (printf format) and returns `code`.
int lope_set_error(int code, const char* fmt, ...);
// Counts one launch of a library kernel (lope_launch_count()).
void lope_count_launch();

// ORACLE TEST INFRASTRUCTURE — GSL subset shim (GSL is not installed here).
// Only gsl_set_error_handler_off, called at /root/reference/proj/src/specfun.cpp:16-19.
#pragma once
typedef void gsl_error_handler_t(const char* reason, const char* file, int line, int gsl_errno);
inline gsl_error_handler_t* gsl_set_error_handler_off() { return nullptr; }

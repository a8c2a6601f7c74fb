// Internal declarations shared by the host (rd_host.cpp) and device (rd_cuda.cu) halves
// of librd.so.  Not part of the C-ABI (see include/rd.h).
#pragma once
#include <cstdint>
#include <vector>

#include "rd.h"

namespace rd {

// Records a thread-local message for rd_last_error() and returns `code`.
int fail(int code, const char *fmt, ...) noexcept;
void clear_error() noexcept;

// The C-ABI never lets an exception out (rd.h "Errors"): every entry point with an int status
// is a function-try-block ending in RD_ABI_CATCH, which maps the in-flight exception to a
// status: std::bad_alloc / std::length_error (a host allocation) -> RD_ENOMEM, anything
// else -> RD_EINVAL with the exception's text.
int abi_exception(const char *who) noexcept;
#define RD_ABI_CATCH(who) \
  catch (...) { return ::rd::abi_exception(who); }

// Number of correct words of length m (Def 4); -1 if m is out of range.
int64_t count_words(int m);
// Correct words as base-4 codes (a=0,b=1,c=2,d=3, row 1 = most significant digit),
// ascending = lexicographic a<b<c<d.
std::vector<uint32_t> word_codes(int m);
// A(G) into A (N*N int16 row-major, RD_INF off the arcs).  OpenMP over rows.
int build_matrix(int m, int16_t *A, int64_t N);
// border = the App. A variant (m = 4): last-row rules of P:594-599, labels 10p(a)+5p(b)-2nd
int build_matrix_variant(int m, int16_t *A, int64_t N, bool border);
// The same arcs as a CSC per q-chunk straight from the successor generator (see rd_host.cpp).
int build_csc_direct(int m, bool border, int nchunks, int Qc, std::vector<int32_t> &colptr,
                     std::vector<uint32_t> &ent, std::vector<int16_t> &diag);

// Packed right operand / pair-major layouts, see DESIGN.md "Data layout".
constexpr int kTile = 128;          // CTA tile (rows and columns of C)
constexpr int kMaxAlpha = 32;
inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

}  // namespace rd

// Host-side big integers for the driver layer (secant bookkeeping on the
// folded determinant, decimal output): declarations of the documented GMP
// mpz ABI, linked against the image's runtime libgmp.so.10 (GMP 6.3.0; the
// image ships no GMP headers).  The reference's driver uses the same library
// for the same host arithmetic (/root/reference/proj/src/secant.cpp).
#pragma once
#include <cstddef>

extern "C" {
typedef struct {
  int _mp_alloc;
  int _mp_size;
  unsigned long* _mp_d;
} hg_mpz_struct;
typedef hg_mpz_struct* hg_mpz_ptr;
typedef const hg_mpz_struct* hg_mpz_srcptr;

void __gmpz_init(hg_mpz_ptr);
void __gmpz_init_set(hg_mpz_ptr, hg_mpz_srcptr);
void __gmpz_init_set_si(hg_mpz_ptr, long);
void __gmpz_clear(hg_mpz_ptr);
void __gmpz_set(hg_mpz_ptr, hg_mpz_srcptr);
void __gmpz_set_si(hg_mpz_ptr, long);
void __gmpz_set_ui(hg_mpz_ptr, unsigned long);
int __gmpz_root(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
unsigned long __gmpz_fdiv_q_ui(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
int __gmpz_set_str(hg_mpz_ptr, const char*, int);
void __gmpz_swap(hg_mpz_ptr, hg_mpz_ptr);
char* __gmpz_get_str(char*, int, hg_mpz_srcptr);
double __gmpz_get_d_2exp(long*, hg_mpz_srcptr);
void __gmpz_add(hg_mpz_ptr, hg_mpz_srcptr, hg_mpz_srcptr);
void __gmpz_sub(hg_mpz_ptr, hg_mpz_srcptr, hg_mpz_srcptr);
void __gmpz_mul(hg_mpz_ptr, hg_mpz_srcptr, hg_mpz_srcptr);
void __gmpz_mul_ui(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
void __gmpz_mul_2exp(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
void __gmpz_neg(hg_mpz_ptr, hg_mpz_srcptr);
void __gmpz_abs(hg_mpz_ptr, hg_mpz_srcptr);
void __gmpz_tdiv_q(hg_mpz_ptr, hg_mpz_srcptr, hg_mpz_srcptr);
void __gmpz_tdiv_q_2exp(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
void __gmpz_fdiv_q(hg_mpz_ptr, hg_mpz_srcptr, hg_mpz_srcptr);
void __gmpz_fdiv_q_2exp(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
void __gmpz_cdiv_q_2exp(hg_mpz_ptr, hg_mpz_srcptr, unsigned long);
void __gmpz_cdiv_q(hg_mpz_ptr, hg_mpz_srcptr, hg_mpz_srcptr);
int __gmpz_cmp(hg_mpz_srcptr, hg_mpz_srcptr);
size_t __gmpz_sizeinbase(hg_mpz_srcptr, int);
void __gmpz_ui_pow_ui(hg_mpz_ptr, unsigned long, unsigned long);
void __gmpz_fac_ui(hg_mpz_ptr, unsigned long);
void __gmpz_setbit(hg_mpz_ptr, unsigned long);
void __gmpz_import(hg_mpz_ptr, size_t, int, size_t, int, size_t, const void*);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, hg_mpz_srcptr);
}

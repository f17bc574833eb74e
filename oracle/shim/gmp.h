/* Minimal GMP 6.x declarations for the oracle build (test infrastructure).
 *
 * The image ships the runtime libgmp.so.10 (GMP 6.3.0) but no development
 * headers.  This file declares, from the documented GMP ABI, only the mpz
 * entry points the reference sources under /root/reference/proj/src call
 * (SURVEY.md §8c lists them) plus a few the oracle restatement uses.  It is
 * linked against /usr/lib/x86_64-linux-gnu/libgmp.so.10 by full path.
 * Not used by the product path.
 */
#ifndef ORACLE_SHIM_GMP_H
#define ORACLE_SHIM_GMP_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef unsigned long mp_bitcnt_t;
typedef long mp_exp_t;

typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

#define GMP_LIMB_BITS 64

void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
int __gmpz_init_set_str(mpz_ptr, const char*, int);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
void __gmpz_set_d(mpz_ptr, double);
int __gmpz_set_str(mpz_ptr, const char*, int);
void __gmpz_swap(mpz_ptr, mpz_ptr);
char* __gmpz_get_str(char*, int, mpz_srcptr);
long __gmpz_get_si(mpz_srcptr);
unsigned long __gmpz_get_ui(mpz_srcptr);
double __gmpz_get_d(mpz_srcptr);
double __gmpz_get_d_2exp(long*, mpz_srcptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_mul_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_addmul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_submul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_fdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
unsigned long __gmpz_fdiv_q_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_cdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_cdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_divexact_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_and(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_ior(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_xor(mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
int __gmpz_cmp_ui(mpz_srcptr, unsigned long);
int __gmpz_cmpabs(mpz_srcptr, mpz_srcptr);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
void __gmpz_ui_pow_ui(mpz_ptr, unsigned long, unsigned long);
void __gmpz_pow_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_setbit(mpz_ptr, mp_bitcnt_t);
int __gmpz_tstbit(mpz_srcptr, mp_bitcnt_t);
void __gmpz_fac_ui(mpz_ptr, unsigned long);
void __gmpz_sqrt(mpz_ptr, mpz_srcptr);
int __gmpz_root(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_gcd(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void*);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, mpz_srcptr);

#define mpz_init __gmpz_init
#define mpz_init_set __gmpz_init_set
#define mpz_init_set_si __gmpz_init_set_si
#define mpz_init_set_ui __gmpz_init_set_ui
#define mpz_init_set_str __gmpz_init_set_str
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_set_si __gmpz_set_si
#define mpz_set_ui __gmpz_set_ui
#define mpz_set_d __gmpz_set_d
#define mpz_set_str __gmpz_set_str
#define mpz_swap __gmpz_swap
#define mpz_get_str __gmpz_get_str
#define mpz_get_si __gmpz_get_si
#define mpz_get_ui __gmpz_get_ui
#define mpz_get_d __gmpz_get_d
#define mpz_get_d_2exp __gmpz_get_d_2exp
#define mpz_add __gmpz_add
#define mpz_add_ui __gmpz_add_ui
#define mpz_sub __gmpz_sub
#define mpz_sub_ui __gmpz_sub_ui
#define mpz_mul __gmpz_mul
#define mpz_mul_si __gmpz_mul_si
#define mpz_mul_ui __gmpz_mul_ui
#define mpz_addmul __gmpz_addmul
#define mpz_submul __gmpz_submul
#define mpz_mul_2exp __gmpz_mul_2exp
#define mpz_neg __gmpz_neg
#define mpz_abs __gmpz_abs
#define mpz_tdiv_q __gmpz_tdiv_q
#define mpz_tdiv_r __gmpz_tdiv_r
#define mpz_tdiv_q_2exp __gmpz_tdiv_q_2exp
#define mpz_fdiv_q __gmpz_fdiv_q
#define mpz_fdiv_r __gmpz_fdiv_r
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_fdiv_q_ui __gmpz_fdiv_q_ui
#define mpz_cdiv_q __gmpz_cdiv_q
#define mpz_cdiv_q_2exp __gmpz_cdiv_q_2exp
#define mpz_divexact_ui __gmpz_divexact_ui
#define mpz_and __gmpz_and
#define mpz_ior __gmpz_ior
#define mpz_xor __gmpz_xor
#define mpz_cmp __gmpz_cmp
#define mpz_cmp_si __gmpz_cmp_si
#define mpz_cmp_ui __gmpz_cmp_ui
#define mpz_cmpabs __gmpz_cmpabs
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_ui_pow_ui __gmpz_ui_pow_ui
#define mpz_pow_ui __gmpz_pow_ui
#define mpz_setbit __gmpz_setbit
#define mpz_tstbit __gmpz_tstbit
#define mpz_fac_ui __gmpz_fac_ui
#define mpz_sqrt __gmpz_sqrt
#define mpz_root __gmpz_root
#define mpz_gcd __gmpz_gcd
#define mpz_import __gmpz_import
#define mpz_export __gmpz_export

#define mpz_sgn(z) ((z)->_mp_size < 0 ? -1 : (z)->_mp_size > 0)

#ifdef __cplusplus
}
#endif

#endif

/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference (hvp, /root/reference/proj) algorithm for the
 * hot path: TFHE gate bootstrapping, identity/private key switching, circuit
 * bootstrapping and the CMUX-Memory trees.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.  Every function cites the reference
 * file:line it restates.  Parity of this restatement is pinned against the reference
 * itself (oracle/_ref/libhvpref.so, built from the reference sources) by
 * tests/test_oracle_pin.py and by the golden fixtures in tests/golden/.
 *
 * Flat layouts are identical to include/vsp_b200.h (TLWE = a[dim] then b;
 * TRLWE = a[N] then b[N]; TRGSW = 2l TRLWE rows).
 */
#ifndef HVP_ORACLE_H
#define HVP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

/* params: "tfhe-80" | "test-det" (params.cpp:31-86); n_override>0 replaces n. */
orc_ctx* orc_ctx_new(const char* name, uint32_t n_override, uint64_t seed);
void orc_ctx_free(orc_ctx* c);
void orc_params(const orc_ctx* c, uint32_t* out14);
/* exact=1 forces schoolbook products at every level (MulBackend::Exact semantics,
 * poly.hpp:15-29) regardless of the parameter set; used to check exact GPU paths. */
void orc_set_exact(orc_ctx* c, int exact);

int orc_keygen(orc_ctx* c, int with_cb);
int orc_import_keys(orc_ctx* c, const uint32_t* lv0, const uint32_t* lv1,
                    const uint32_t* lv2, const uint32_t* bk1, const uint64_t* bk2,
                    const uint32_t* ksk, const uint32_t* pks_negs,
                    const uint32_t* pks_id, int has_cb);
int orc_export_sk(const orc_ctx* c, uint32_t* lv0, uint32_t* lv1, uint32_t* lv2);
int orc_export_bk1(const orc_ctx* c, uint32_t* out);
int orc_export_bk2(const orc_ctx* c, uint64_t* out);
size_t orc_ksk_words(const orc_ctx* c);
int orc_export_ksk(const orc_ctx* c, uint32_t* out);
size_t orc_pks_words(const orc_ctx* c);
int orc_export_pks(const orc_ctx* c, int which, uint32_t* out);

int orc_tlwe_encrypt(orc_ctx* c, int m, uint32_t* out);
uint32_t orc_tlwe_phase(const orc_ctx* c, const uint32_t* ct, int level);
int orc_trlwe_encrypt(orc_ctx* c, const uint32_t* bits, double alpha, uint32_t* out);
uint32_t orc_trlwe_phase_at(const orc_ctx* c, const uint32_t* ct, uint32_t k);
int orc_trgsw_encrypt(orc_ctx* c, int m, double alpha, uint32_t* out);

int orc_hom_gate(orc_ctx* c, int kind, const uint32_t* in, int nin, uint32_t* out);
int orc_hom_gate_batch(orc_ctx* c, const int* kinds, const uint32_t* in, uint32_t* out,
                       size_t G, unsigned threads);
int orc_gate_bootstrap(orc_ctx* c, const uint32_t* in, uint32_t* out);
int orc_bootstrap_to_trlwe(orc_ctx* c, const uint32_t* in, uint32_t* out);
int orc_blind_rotate_lvl2(orc_ctx* c, const uint32_t* in, const uint64_t* testvec,
                          uint64_t* out);
/* T level-2 blind rotations with test vectors b = h[t]/2 on `threads` threads. */
int orc_blind_rotate_lvl2_batch(orc_ctx* c, const uint32_t* in, const uint64_t* h,
                                uint64_t* out, size_t T, unsigned threads);
int orc_identity_key_switch(orc_ctx* c, const uint32_t* in, uint32_t* out);
int orc_sample_extract(orc_ctx* c, const uint32_t* trlwe, uint32_t k, uint32_t* out);
int orc_external_product(orc_ctx* c, const uint32_t* trgsw, const uint32_t* trlwe,
                         uint32_t* out);
int orc_external_product_lvl2(orc_ctx* c, const uint64_t* trgsw, const uint64_t* trlwe,
                              uint64_t* out);
int orc_cmux(orc_ctx* c, const uint32_t* sel, const uint32_t* c1, const uint32_t* c0,
             uint32_t* out);
int orc_hom_mux_no_se_iks(orc_ctx* c, const uint32_t* sel, const uint32_t* a,
                          const uint32_t* b, uint32_t* out);
int orc_circuit_bootstrap(orc_ctx* c, const uint32_t* in, uint32_t* out);
int orc_private_key_switch(orc_ctx* c, const uint64_t* in, int which, uint32_t* out);
int orc_trgsw_not(orc_ctx* c, const uint32_t* in, uint32_t* out);

int orc_ram_cycle(orc_ctx* c, uint32_t v, uint32_t w, uint32_t* ram,
                  const uint32_t* addr, const uint32_t* wflag, const uint32_t* wdata,
                  uint32_t* readout);
int orc_rom_read(orc_ctx* c, uint32_t depth_bytes, const uint32_t* luts,
                 uint32_t nluts, const uint32_t* addr, uint32_t vrom, uint32_t* out);
int orc_encrypt_ram(orc_ctx* c, const uint8_t* image, uint32_t v, uint32_t w,
                    int trivial, uint32_t* out);
int orc_decrypt_ram(const orc_ctx* c, const uint32_t* ram, uint32_t v, uint32_t w,
                    uint8_t* image);
uint32_t orc_rom_luts(const orc_ctx* c, uint32_t depth_bytes);
int orc_encrypt_rom(orc_ctx* c, const uint8_t* image, uint32_t depth_bytes, int trivial,
                    uint32_t* out);

void orc_counters(uint64_t* out5);
void orc_counters_reset(void);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif

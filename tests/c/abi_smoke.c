/* Plain-C consumer of libmpsf.so (no Python, no CUDA headers): what a non-Python binding of
 * the reference would compile against.  Uses only entry points that need no device: the
 * version, the status strings and the host-side trace renderer. */
#include <stdio.h>
#include <string.h>

#include "mpsf.h"

int main(void) {
  if (mpsf_version() != MPSF_ABI_VERSION) return 1;
  if (!mpsf_strerror(MPSF_E_NO_CHANNEL) || !strlen(mpsf_strerror(MPSF_E_NO_CHANNEL))) return 2;
  mpsf_fault_entry e[2];
  memset(e, 0, sizeof e);
  e[0].va = 0x1000; e[0].channel = 0; e[0].engine = 0; e[0].access = 1; e[0].kind = 0; e[0].flags = 1;
  e[1].va = 0;      e[1].channel = 1; e[1].engine = 1; e[1].access = 0; e[1].kind = 2; e[1].flags = 1;
  mpsf_out_record o[2];
  memset(o, 0, sizeof o);
  o[0].scenario = 0;  o[0].verdict = 2 | (1 << 2) | 0x40; o[0].client = 0;   /* isolated M1, replayable */
  o[1].scenario = 24; o[1].verdict = 3 | 0x40;            o[1].client = 0;   /* parse-time fatal */
  const char* chans[2] = {"c1.sm", "c1.ce"};
  const char* clients[1] = {"c1"};
  mpsf_render_params p;
  memset(&p, 0, sizeof p);
  p.t_drain = 42; p.m1_us = 131; p.m2_us = 2780; p.m3_us = 1700;
  p.parts = MPSF_RENDER_TOP | MPSF_RENDER_DRAIN;
  p.channel_names = chans; p.n_channels = 2; p.client_names = clients; p.n_clients = 1;
  const int64_t need = mpsf_render_trace(e, o, 2, &p, NULL, 0);
  if (need <= 0) return 3;
  char buf[4096];
  if (need >= (int64_t)sizeof buf) return 4;
  if (mpsf_render_trace(e, o, 2, &p, buf, sizeof buf) != need) return 5;
  buf[need] = 0;
  fputs(buf, stdout);
  return 0;
}

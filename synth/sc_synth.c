/* Seeded synthetic inputs of the five BASELINE.json configurations (SURVEY.md
 * §8d) -- bench / test input generation only, kept out of the product library
 * (libslicecraft_b200.so) and out of the oracle, so that both bench arms (the
 * B200 path and the reference CPU path) consume identical bytes from a library
 * that is neither.
 *
 * Luma: base gradient g = (x*M/(W-1) + y*M/(H-1)) / 2; 128x128 blocks with the
 * lattice drifted by 4 px per frame; a block is noise (H(seed,f,x,y) mod M+1)
 * with probability textured_pct %, else the gradient; mode 1 is config 2's
 * flat / gradient / noise thirds.  Integer-only, reproducible everywhere.
 * Times: lognormal(0, sigma) by Box-Muller from two hash uniforms, rounded to
 * float then widened (libm exp/log/cos). */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <unistd.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline uint64_t H4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return mix64(mix64(mix64(seed ^ mix64(a)) ^ b) ^ (c * 0x2545f4914f6cdd1dull));
}

typedef struct {
  uint64_t seed;
  int W, H, bits, first, pct, mode, f0, f1;
  void* out;
} Job;

static void* luma_frames(void* arg) {
  const Job* j = (const Job*)arg;
  const int bps = j->bits <= 8 ? 1 : 2;
  const uint32_t M = (1u << j->bits) - 1u;
  const size_t fbytes = (size_t)j->W * j->H * bps;
  for (int fi = j->f0; fi < j->f1; ++fi) {
    const int f = j->first + fi;
    unsigned char* base = (unsigned char*)j->out + (size_t)fi * fbytes;
    for (int y = 0; y < j->H; ++y) {
      const int by = y / 128;
      for (int x = 0; x < j->W; ++x) {
        const int bx = (x + 4 * f) / 128;
        const uint32_t g = (uint32_t)(((uint64_t)x * M / (uint64_t)(j->W > 1 ? j->W - 1 : 1) +
                                       (uint64_t)y * M / (uint64_t)(j->H > 1 ? j->H - 1 : 1)) / 2);
        uint32_t v;
        const uint64_t hb = H4(j->seed, (uint64_t)bx, (uint64_t)by, 0);
        if (j->mode == 1) {
          const uint32_t cls = (uint32_t)(H4(j->seed, (uint64_t)bx, (uint64_t)by, 1) % 3);
          if (cls == 0) v = (uint32_t)(H4(j->seed, (uint64_t)bx, (uint64_t)by, 2) % (M + 1));
          else if (cls == 1) v = g;
          else v = (uint32_t)(H4(j->seed, (uint64_t)f, (uint64_t)x, (uint64_t)y) % (M + 1));
        } else if ((int)(hb % 100) < j->pct) {
          v = (uint32_t)(H4(j->seed, (uint64_t)f, (uint64_t)x, (uint64_t)y) % (M + 1));
        } else {
          v = g;
        }
        if (bps == 1) base[(size_t)y * j->W + x] = (unsigned char)v;
        else ((uint16_t*)base)[(size_t)y * j->W + x] = (uint16_t)v;
      }
    }
  }
  return NULL;
}

/* n_frames frames starting at frame index first_frame, packed (stride W*H*bps).
 * Returns 0, or -1 on bad arguments. */
int sc_synth_luma(uint64_t seed, int32_t W, int32_t H, int32_t bit_depth, int32_t frames,
                  int32_t first_frame, int32_t pct, int32_t mode, void* out) {
  if (!out || W < 1 || H < 1 || frames < 1 || bit_depth < 1 || bit_depth > 16) return -1;
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > 32) nt = 32;
  if (nt > frames) nt = frames;
  pthread_t th[32];
  Job jobs[32];
  for (int t = 0; t < nt; ++t) {
    Job j = {seed, W, H, bit_depth, first_frame, pct, mode,
             (int)((int64_t)frames * t / nt), (int)((int64_t)frames * (t + 1) / nt), out};
    jobs[t] = j;
    pthread_create(&th[t], NULL, luma_frames, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  return 0;
}

int sc_synth_times(uint64_t seed, int32_t tag, int32_t cells, double sigma, double* out) {
  if (!out || cells < 1) return -1;
  for (int i = 0; i < cells; ++i) {
    const double u1 = ((H4(seed, 0x71e5ull + (uint64_t)tag, (uint64_t)i, 1) >> 11) + 1) *
                      (1.0 / 9007199254740992.0);
    const double u2 = (H4(seed, 0x71e5ull + (uint64_t)tag, (uint64_t)i, 2) >> 11) *
                      (1.0 / 9007199254740992.0);
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    out[i] = (double)(float)exp(sigma * z);
  }
  return 0;
}

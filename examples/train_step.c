/* train_step.c -- the TawPipe step driven from C through include/tawpipe.h alone (no Python in the process).
 *
 * One process per GPU.  World size 1 by default; for a multi-rank job set TAWPIPE_RANK, TAWPIPE_WORLD, TAWPIPE_GROUP
 * (group size G) and TAWPIPE_ID_FILE in each process's environment: rank 0 writes the 128-byte NCCL unique id
 * (tawpipe_get_unique_id) to that file, the other ranks wait for it, and every rank calls
 * tawpipe_bootstrap(rank, world, device = rank, id) -- no torch.distributed involved.
 *
 *   train_step L H n_h I V S B n_micro dtype steps tokens.i32 [weights.f32|-] [shard_out.f32]
 *
 *   tokens.i32   steps x [n_micro][B][S+1] int32 (the layout tawpipe_step takes: inputs x[0..S-1],
 *                targets x[1..S])
 *   weights.f32  optional canonical full model for tawpipe_load ("-": the library's seeded device init)
 *   shard_out    optional: this rank's owned fp32 master after the last step (tawpipe_shard)
 *
 * Prints "loss <step> <value>" per step (the global mean loss tawpipe_step returns).  Exit code: 0, or 2 on a
 * usage / file error, or 1 with tawpipe_last_error() on a library error.
 *
 * Build (the library's own NCCL dependency is found through its RUNPATH):
 *   gcc -O2 -I include examples/train_step.c -L paper_2511_09741_b200 -ltawpipe \
 *       -Wl,-rpath,$PWD/paper_2511_09741_b200 -Wl,--allow-shlib-undefined -o train_step
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "tawpipe.h"

static void* read_file(const char* path, long* bytes) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  void* p = malloc((size_t)*bytes);
  if (p && fread(p, 1, (size_t)*bytes, f) != (size_t)*bytes) {
    free(p);
    p = NULL;
  }
  fclose(f);
  return p;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

/* rank 0 publishes the NCCL unique id through a file (written under a temporary name, then renamed, so a reader
 * never sees a partial id); the other ranks poll for it for up to 60 s */
static int exchange_id(int rank, const char* path, char id[128]) {
  if (rank == 0) {
    if (tawpipe_get_unique_id(id) != TAWPIPE_OK) return -1;
    char tmp[4096];
    snprintf(tmp, sizeof(tmp), "%s.tmp", path);
    FILE* f = fopen(tmp, "wb");
    if (!f || fwrite(id, 1, 128, f) != 128) return -1;
    fclose(f);
    return rename(tmp, path);
  }
  for (int i = 0; i < 6000; ++i) {
    FILE* f = fopen(path, "rb");
    if (f) {
      const size_t n = fread(id, 1, 128, f);
      fclose(f);
      if (n == 128) return 0;
    }
    usleep(10000);
  }
  return -1;
}

static int fail(const char* what) {
  fprintf(stderr, "%s: %s\n", what, tawpipe_last_error());
  return 1;
}

int main(int argc, char** argv) {
  if (argc < 12) {
    fprintf(stderr, "usage: %s L H n_h I V S B n_micro dtype steps tokens.i32 [weights.f32|-] [shard_out.f32]\n",
            argv[0]);
    return 2;
  }
  const int L = atoi(argv[1]), n_micro = atoi(argv[8]), steps = atoi(argv[10]);
  tawpipe_dims d = {0};
  d.hidden = atoi(argv[2]);
  d.heads = atoi(argv[3]);
  d.ffn = atoi(argv[4]);
  d.vocab = atoi(argv[5]);
  d.seq = atoi(argv[6]);
  d.micro_bs = atoi(argv[7]);
  d.dtype = atoi(argv[9]);
  d.ckpt = 0;
  d.schedule = TAWPIPE_GWPS;
  d.lr = 1e-3f;   /* the defaults of the Python binding's ModelDims (LLaMA-2 conventions, R1 / R10) */
  d.beta1 = 0.9f;
  d.beta2 = 0.95f;
  d.adam_eps = 1e-8f;
  d.weight_decay = 0.1f;
  d.rms_eps = 1e-5f;
  d.rope_theta = 10000.0f;
  d.seed = 1234;

  long tok_bytes = 0;
  int32_t* tokens = (int32_t*)read_file(argv[11], &tok_bytes);
  const long per_step = (long)n_micro * d.micro_bs * (d.seq + 1);
  if (!tokens || tok_bytes != (long)sizeof(int32_t) * per_step * steps) {
    fprintf(stderr, "tokens file %s: expected %ld int32\n", argv[11], per_step * steps);
    return 2;
  }

  const int rank = env_int("TAWPIPE_RANK", 0), world = env_int("TAWPIPE_WORLD", 1);
  const int group = env_int("TAWPIPE_GROUP", world);
  char id[128];
  memset(id, 0, sizeof(id));
  if (world > 1) {
    const char* id_file = getenv("TAWPIPE_ID_FILE");
    if (!id_file || exchange_id(rank, id_file, id) != 0) {
      fprintf(stderr, "rank %d: NCCL unique id exchange through TAWPIPE_ID_FILE failed\n", rank);
      return 2;
    }
  }
  if (tawpipe_bootstrap(rank, world, rank, world > 1 ? id : NULL) != TAWPIPE_OK) return fail("tawpipe_bootstrap");
  if (tawpipe_init(world, group, L, &d, n_micro) != TAWPIPE_OK) return fail("tawpipe_init");
  if (argc > 12 && argv[12][0] != '-') {
    long w_bytes = 0;
    float* w = (float*)read_file(argv[12], &w_bytes);
    if (!w) {
      fprintf(stderr, "cannot read %s\n", argv[12]);
      return 2;
    }
    if (tawpipe_load(w, w_bytes / (long)sizeof(float)) != TAWPIPE_OK) return fail("tawpipe_load");
    free(w);
  }
  for (int s = 0; s < steps; ++s) {
    const float loss = tawpipe_step(tokens + (long)s * per_step);
    if (isnan(loss)) return fail("tawpipe_step");
    printf("loss %d %.9g\n", s, loss);
  }
  if (argc > 13) {
    const int64_t n = tawpipe_shard_elems();
    float* out = (float*)malloc((size_t)n * sizeof(float));
    if (!out || tawpipe_shard(out) != n) return fail("tawpipe_shard");
    FILE* f = fopen(argv[13], "wb");
    if (!f || fwrite(out, sizeof(float), (size_t)n, f) != (size_t)n) {
      fprintf(stderr, "cannot write %s\n", argv[13]);
      return 2;
    }
    fclose(f);
    free(out);
  }
  tawpipe_finalize();
  free(tokens);
  return 0;
}

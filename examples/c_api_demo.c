/* The drop-in boundary from plain C (no Python, no torch): include/mdrt.h + libmdrt.so.
 *
 * One flat 10 m x 10 m ground plane (2 triangles) as terrain, one 0.3 m box body
 * hovering over it, one 9x7 camera at 1 m height looking straight down (the
 * reference's analytic test, test_render.py:23-32), 2 envs whose box sits at a
 * different height. The centre pixel must read the box top (env 0) and the
 * ground (env 1); misses read exactly float32(d_max).
 *
 *   gcc -O2 -I include examples/c_api_demo.c -o build/c_api_demo \
 *       -L paper_2602_03002_b200 -lmdrt -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2602_03002_b200
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "mdrt.h"

#define CHECK(call)                                                                      \
    do {                                                                                 \
        int rc_ = (call);                                                                \
        if (rc_ != MDRT_OK) {                                                            \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, mdrt_last_error());     \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

int main(void) {
    int32_t ndev = 0;
    CHECK(mdrt_device_count(&ndev));
    if (ndev < 1) {
        fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    mdrt_ctx* ctx = NULL;
    CHECK(mdrt_create(0, &ctx));

    /* terrain: z = 0 plane */
    const double tv[] = {-5, -5, 0, 5, -5, 0, 5, 5, 0, -5, 5, 0};
    const int64_t tf[] = {0, 1, 2, 0, 2, 3};
    CHECK(mdrt_set_terrain(ctx, tv, 4, tf, 2));

    /* body: axis-aligned 0.3 m cube centred on its local origin */
    double bv[8 * 3];
    for (int i = 0; i < 8; ++i) {
        bv[3 * i + 0] = (i & 1) ? 0.15 : -0.15;
        bv[3 * i + 1] = (i & 2) ? 0.15 : -0.15;
        bv[3 * i + 2] = (i & 4) ? 0.15 : -0.15;
    }
    const int64_t bf[] = {0, 2, 1, 1, 2, 3, 4, 5, 6, 5, 7, 6, 0, 1, 4, 1, 5, 4,
                          2, 6, 3, 3, 6, 7, 0, 4, 2, 2, 4, 6, 1, 3, 5, 3, 7, 5};
    int32_t body = -1;
    CHECK(mdrt_add_body(ctx, bv, 8, bf, 12, &body));

    /* camera: 1 m above the origin looking down (+z forward = world -z; +y down = world -y) */
    const double hfov = 70.0, vfov = 55.0, dmax = 5.0;
    const int32_t parent = -1;
    const double mpos[] = {0, 0, 1};
    const double mrot[] = {0.0, 1.0, 0.0, 0.0};   /* wxyz: 180 deg about x */
    CHECK(mdrt_set_cameras(ctx, 1, 9, 7, &hfov, &vfov, &dmax, &parent, mpos, mrot));
    CHECK(mdrt_commit(ctx));

    /* two envs: box top at z = 0.5 (env 0) and far away (env 1) */
    const int N = 2, W = 9, H = 7;
    float hpos[2 * 3] = {0, 0, 0.35f, 50, 50, 0.35f};
    float hrot[2 * 4] = {1, 0, 0, 0, 1, 0, 0, 0};
    float *dpos, *drot, *dout;
    if (cudaMalloc((void**)&dpos, sizeof hpos) || cudaMalloc((void**)&drot, sizeof hrot) ||
        cudaMalloc((void**)&dout, sizeof(float) * N * W * H)) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(dpos, hpos, sizeof hpos, cudaMemcpyHostToDevice);
    cudaMemcpy(drot, hrot, sizeof hrot, cudaMemcpyHostToDevice);

    mdrt_step_args a;
    memset(&a, 0, sizeof a);
    a.num_envs = N;
    a.flags = MDRT_EARLY_TERMINATION;
    a.body_pos = dpos;
    a.body_rot = drot;
    a.ray_envs = 1;
    a.out = dout;
    CHECK(mdrt_render(ctx, &a, NULL));
    float out[2 * 7 * 9];
    if (cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost)) {
        fprintf(stderr, "cudaMemcpy failed\n");
        return 1;
    }
    const float centre0 = out[0 * H * W + 3 * W + 4], centre1 = out[1 * H * W + 3 * W + 4];
    printf("centre range: env 0 %.6f m (box top, expect 0.5), env 1 %.6f m (ground, expect 1.0)\n", centre0, centre1);
    int ok = fabsf(centre0 - 0.5f) < 1e-5f && fabsf(centre1 - 1.0f) < 1e-5f;

    /* argument errors come back as MDRT_EINVAL with a message, as the reference raises ValueError */
    a.num_envs = 0;
    int rc = mdrt_render(ctx, &a, NULL);
    printf("num_envs = 0 -> %d (%s)\n", rc, mdrt_last_error());
    ok = ok && rc == MDRT_EINVAL;

    CHECK(mdrt_destroy(ctx));
    cudaFree(dpos);
    cudaFree(drot);
    cudaFree(dout);
    printf(ok ? "c_api_demo ok\n" : "c_api_demo FAILED\n");
    return ok ? 0 : 1;
}

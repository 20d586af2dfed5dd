// Compile as OpenCL with this prelude:
//   #define KERNEL __kernel
//   #define GLOBAL __global
//   #define LOCAL __local
//   #define GROUP_ID(n) ((int) get_group_id(n))
//   #define LOCAL_ID(n) ((int) get_local_id(n))
//   #define BARRIER() barrier(CLK_LOCAL_MEM_FENCE)
//   typedef float4 vec4f;

// kernel: fused_r_s
// launch: groups = Ne, lanes per group = 3 x 3
KERNEL void fused_r_s(int Ne, float p0, float Rgas, float gam, GLOBAL const vec4f* restrict q, GLOBAL vec4f* restrict rhsq, GLOBAL const float* restrict D, GLOBAL const float* restrict g, GLOBAL const float* restrict Jinv)
{
    const int e = GROUP_ID(0);
    const int i = LOCAL_ID(0);
    const int j = LOCAL_ID(1);
    float flxu_r;
    float flx1_r;
    float flx2_r;
    float flx3_r;
    float flx4_r;
    float flx5_r;
    float flx6_r;
    float flx7_r;
    float flx8_r;
    float flxu_s;
    float flx1_s;
    float flx2_s;
    float flx3_s;
    float flx4_s;
    float flx5_s;
    float flx6_s;
    float flx7_s;
    float flx8_s;
    float tflxu_s;
    float tflx1_s;
    float tflx2_s;
    float tflx3_s;
    float tflx4_s;
    float tflx5_s;
    float tflx6_s;
    float tflx7_s;
    float tflx8_s;
    LOCAL float D_pf[9];
    for (int D_f0 = 0; D_f0 < 3; ++D_f0)
    {
        for (int D_f1 = 0; D_f1 < 3; ++D_f1)
        {
            if (LOCAL_ID(0) == 0 && LOCAL_ID(1) == 0) {
                D_pf[(D_f1) * 3 + D_f0] = D[(D_f1) * 3 + D_f0];  // D_pf_fetch
            }
        }
    }
    for (int k = 0; k < 3; ++k)
    {
        BARRIER();
        tflxu_s = g[(((((e) * 3 + 2) * 3 + 0) * 3 + k) * 3 + j) * 3 + i] * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 + g[(((((e) * 3 + 2) * 3 + 1) * 3 + k) * 3 + j) * 3 + i] * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 + g[(((((e) * 3 + 2) * 3 + 2) * 3 + k) * 3 + j) * 3 + i] * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3;  // i43_tflxu_s
        tflx1_s = tflxu_s;  // i44_tflx1_s
        tflx2_s = g[(((((e) * 3 + 2) * 3 + 0) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 / p0, gam)) + g[(((((e) * 3 + 2) * 3 + 1) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0)) + g[(((((e) * 3 + 2) * 3 + 2) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0));  // i45_tflx2_s
        tflx3_s = g[(((((e) * 3 + 2) * 3 + 0) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0)) + g[(((((e) * 3 + 2) * 3 + 1) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 / p0, gam)) + g[(((((e) * 3 + 2) * 3 + 2) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0));  // i46_tflx3_s
        tflx4_s = g[(((((e) * 3 + 2) * 3 + 0) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0)) + g[(((((e) * 3 + 2) * 3 + 1) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0)) + g[(((((e) * 3 + 2) * 3 + 2) * 3 + k) * 3 + j) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 / p0, gam));  // i47_tflx4_s
        tflx5_s = tflxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0);  // i48_tflx5_s
        tflx6_s = tflxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0);  // i49_tflx6_s
        tflx7_s = tflxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0);  // i50_tflx7_s
        tflx8_s = tflxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0);  // i51_tflx8_s
        for (int n = 0; n < 3; ++n)
        {
            flxu_r = g[(((((e) * 3 + 0) * 3 + 0) * 3 + k) * 3 + j) * 3 + n] * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 + g[(((((e) * 3 + 0) * 3 + 1) * 3 + k) * 3 + j) * 3 + n] * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 + g[(((((e) * 3 + 0) * 3 + 2) * 3 + k) * 3 + j) * 3 + n] * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3;  // i13_flxu_r
            flx1_r = flxu_r;  // i14_flx1_r
            flx2_r = g[(((((e) * 3 + 0) * 3 + 0) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s0 / p0, gam)) + g[(((((e) * 3 + 0) * 3 + 1) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0)) + g[(((((e) * 3 + 0) * 3 + 2) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0));  // i15_flx2_r
            flx3_r = g[(((((e) * 3 + 0) * 3 + 0) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0)) + g[(((((e) * 3 + 0) * 3 + 1) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s0 / p0, gam)) + g[(((((e) * 3 + 0) * 3 + 2) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0));  // i16_flx3_r
            flx4_r = g[(((((e) * 3 + 0) * 3 + 0) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0)) + g[(((((e) * 3 + 0) * 3 + 1) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0)) + g[(((((e) * 3 + 0) * 3 + 2) * 3 + k) * 3 + j) * 3 + n] * (q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s0 / p0, gam));  // i17_flx4_r
            flx5_r = flxu_r * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s0 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0);  // i18_flx5_r
            flx6_r = flxu_r * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0);  // i19_flx6_r
            flx7_r = flxu_r * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0);  // i20_flx7_r
            flx8_r = flxu_r * q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0);  // i21_flx8_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx1_r;  // i22_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx2_r;  // i23_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx3_r;  // i24_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx4_r;  // i25_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx5_r;  // i26_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx6_r;  // i27_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx7_r;  // i28_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx8_r;  // i29_rhsq_r
            flxu_s = g[(((((e) * 3 + 1) * 3 + 0) * 3 + k) * 3 + n) * 3 + i] * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 + g[(((((e) * 3 + 1) * 3 + 1) * 3 + k) * 3 + n) * 3 + i] * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 + g[(((((e) * 3 + 1) * 3 + 2) * 3 + k) * 3 + n) * 3 + i] * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3;  // i13_flxu_s
            flx1_s = flxu_s;  // i14_flx1_s
            flx2_s = g[(((((e) * 3 + 1) * 3 + 0) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s0 / p0, gam)) + g[(((((e) * 3 + 1) * 3 + 1) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0)) + g[(((((e) * 3 + 1) * 3 + 2) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0));  // i15_flx2_s
            flx3_s = g[(((((e) * 3 + 1) * 3 + 0) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0)) + g[(((((e) * 3 + 1) * 3 + 1) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s0 / p0, gam)) + g[(((((e) * 3 + 1) * 3 + 2) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0));  // i16_flx3_s
            flx4_s = g[(((((e) * 3 + 1) * 3 + 0) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0)) + g[(((((e) * 3 + 1) * 3 + 1) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0)) + g[(((((e) * 3 + 1) * 3 + 2) * 3 + k) * 3 + n) * 3 + i] * (q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3 * q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0) + p0 * pow(Rgas * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s0 / p0, gam));  // i17_flx4_s
            flx5_s = flxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s0 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0);  // i18_flx5_s
            flx6_s = flxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s1 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0);  // i19_flx6_s
            flx7_s = flxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s2 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0);  // i20_flx7_s
            flx8_s = flxu_s * q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s3 * (1.0f / q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0);  // i21_flx8_s
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx1_s;  // i22_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx2_s;  // i23_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx3_s;  // i24_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx4_s;  // i25_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx5_s;  // i26_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx6_s;  // i27_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx7_s;  // i28_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + j] * flx8_s;  // i29_rhsq_s
        }
        for (int m = 0; m < 3; ++m)
        {
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx1_s;  // i52_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx2_s;  // i53_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx3_s;  // i54_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx4_s;  // i55_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx5_s;  // i56_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx6_s;  // i57_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx7_s;  // i58_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx8_s;  // i59_rhsq_s
        }
    }
}

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
    float rho_r;
    float rhoinv_r;
    float u1_r;
    float u2_r;
    float u3_r;
    float th_r;
    float qt1_r;
    float qt2_r;
    float qt3_r;
    float p_r;
    float g1_r;
    float g2_r;
    float g3_r;
    float flxu_r;
    float flx1_r;
    float flx2_r;
    float flx3_r;
    float flx4_r;
    float flx5_r;
    float flx6_r;
    float flx7_r;
    float flx8_r;
    float rho_s;
    float rhoinv_s;
    float u1_s;
    float u2_s;
    float u3_s;
    float th_s;
    float qt1_s;
    float qt2_s;
    float qt3_s;
    float p_s;
    float g1_s;
    float g2_s;
    float g3_s;
    float flxu_s;
    float flx1_s;
    float flx2_s;
    float flx3_s;
    float flx4_s;
    float flx5_s;
    float flx6_s;
    float flx7_s;
    float flx8_s;
    float rhop_s;
    float rhopinv_s;
    float v1_s;
    float v2_s;
    float v3_s;
    float thp_s;
    float qp1_s;
    float qp2_s;
    float qp3_s;
    float pp_s;
    float h1_s;
    float h2_s;
    float h3_s;
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
        rhop_s = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0;  // i30_rhop_s
        v1_s = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1;  // i31_v1_s
        v2_s = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2;  // i32_v2_s
        v3_s = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3;  // i33_v3_s
        thp_s = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0;  // i34_thp_s
        qp1_s = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1;  // i35_qp1_s
        qp2_s = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2;  // i36_qp2_s
        qp3_s = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3;  // i37_qp3_s
        rhopinv_s = 1.0f / rhop_s;  // i38_rhopinv_s
        pp_s = p0 * pow(Rgas * thp_s / p0, gam);  // i39_pp_s
        h1_s = g[(((((e) * 3 + 2) * 3 + 0) * 3 + k) * 3 + j) * 3 + i];  // i40_h1_s
        h2_s = g[(((((e) * 3 + 2) * 3 + 1) * 3 + k) * 3 + j) * 3 + i];  // i41_h2_s
        h3_s = g[(((((e) * 3 + 2) * 3 + 2) * 3 + k) * 3 + j) * 3 + i];  // i42_h3_s
        tflxu_s = h1_s * v1_s + h2_s * v2_s + h3_s * v3_s;  // i43_tflxu_s
        tflx1_s = tflxu_s;  // i44_tflx1_s
        tflx2_s = h1_s * (v1_s * v1_s * rhopinv_s + pp_s) + h2_s * (v1_s * v2_s * rhopinv_s) + h3_s * (v1_s * v3_s * rhopinv_s);  // i45_tflx2_s
        tflx3_s = h1_s * (v2_s * v1_s * rhopinv_s) + h2_s * (v2_s * v2_s * rhopinv_s + pp_s) + h3_s * (v2_s * v3_s * rhopinv_s);  // i46_tflx3_s
        tflx4_s = h1_s * (v3_s * v1_s * rhopinv_s) + h2_s * (v3_s * v2_s * rhopinv_s) + h3_s * (v3_s * v3_s * rhopinv_s + pp_s);  // i47_tflx4_s
        tflx5_s = tflxu_s * thp_s * rhopinv_s;  // i48_tflx5_s
        tflx6_s = tflxu_s * qp1_s * rhopinv_s;  // i49_tflx6_s
        tflx7_s = tflxu_s * qp2_s * rhopinv_s;  // i50_tflx7_s
        tflx8_s = tflxu_s * qp3_s * rhopinv_s;  // i51_tflx8_s
        for (int n = 0; n < 3; ++n)
        {
            rho_r = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s0;  // i00_rho_r
            u1_r = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s1;  // i01_u1_r
            u2_r = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s2;  // i02_u2_r
            u3_r = q[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + n].s3;  // i03_u3_r
            th_r = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s0;  // i04_th_r
            qt1_r = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s1;  // i05_qt1_r
            qt2_r = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s2;  // i06_qt2_r
            qt3_r = q[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + n].s3;  // i07_qt3_r
            rhoinv_r = 1.0f / rho_r;  // i08_rhoinv_r
            p_r = p0 * pow(Rgas * th_r / p0, gam);  // i09_p_r
            g1_r = g[(((((e) * 3 + 0) * 3 + 0) * 3 + k) * 3 + j) * 3 + n];  // i10_g1_r
            g2_r = g[(((((e) * 3 + 0) * 3 + 1) * 3 + k) * 3 + j) * 3 + n];  // i11_g2_r
            g3_r = g[(((((e) * 3 + 0) * 3 + 2) * 3 + k) * 3 + j) * 3 + n];  // i12_g3_r
            flxu_r = g1_r * u1_r + g2_r * u2_r + g3_r * u3_r;  // i13_flxu_r
            flx1_r = flxu_r;  // i14_flx1_r
            flx2_r = g1_r * (u1_r * u1_r * rhoinv_r + p_r) + g2_r * (u1_r * u2_r * rhoinv_r) + g3_r * (u1_r * u3_r * rhoinv_r);  // i15_flx2_r
            flx3_r = g1_r * (u2_r * u1_r * rhoinv_r) + g2_r * (u2_r * u2_r * rhoinv_r + p_r) + g3_r * (u2_r * u3_r * rhoinv_r);  // i16_flx3_r
            flx4_r = g1_r * (u3_r * u1_r * rhoinv_r) + g2_r * (u3_r * u2_r * rhoinv_r) + g3_r * (u3_r * u3_r * rhoinv_r + p_r);  // i17_flx4_r
            flx5_r = flxu_r * th_r * rhoinv_r;  // i18_flx5_r
            flx6_r = flxu_r * qt1_r * rhoinv_r;  // i19_flx6_r
            flx7_r = flxu_r * qt2_r * rhoinv_r;  // i20_flx7_r
            flx8_r = flxu_r * qt3_r * rhoinv_r;  // i21_flx8_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx1_r;  // i22_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx2_r;  // i23_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx3_r;  // i24_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx4_r;  // i25_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx5_r;  // i26_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx6_r;  // i27_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx7_r;  // i28_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n) * 3 + i] * flx8_r;  // i29_rhsq_r
            rho_s = q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s0;  // i00_rho_s
            u1_s = q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s1;  // i01_u1_s
            u2_s = q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s2;  // i02_u2_s
            u3_s = q[((((e) * 2 + 0) * 3 + k) * 3 + n) * 3 + i].s3;  // i03_u3_s
            th_s = q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s0;  // i04_th_s
            qt1_s = q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s1;  // i05_qt1_s
            qt2_s = q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s2;  // i06_qt2_s
            qt3_s = q[((((e) * 2 + 1) * 3 + k) * 3 + n) * 3 + i].s3;  // i07_qt3_s
            rhoinv_s = 1.0f / rho_s;  // i08_rhoinv_s
            p_s = p0 * pow(Rgas * th_s / p0, gam);  // i09_p_s
            g1_s = g[(((((e) * 3 + 1) * 3 + 0) * 3 + k) * 3 + n) * 3 + i];  // i10_g1_s
            g2_s = g[(((((e) * 3 + 1) * 3 + 1) * 3 + k) * 3 + n) * 3 + i];  // i11_g2_s
            g3_s = g[(((((e) * 3 + 1) * 3 + 2) * 3 + k) * 3 + n) * 3 + i];  // i12_g3_s
            flxu_s = g1_s * u1_s + g2_s * u2_s + g3_s * u3_s;  // i13_flxu_s
            flx1_s = flxu_s;  // i14_flx1_s
            flx2_s = g1_s * (u1_s * u1_s * rhoinv_s + p_s) + g2_s * (u1_s * u2_s * rhoinv_s) + g3_s * (u1_s * u3_s * rhoinv_s);  // i15_flx2_s
            flx3_s = g1_s * (u2_s * u1_s * rhoinv_s) + g2_s * (u2_s * u2_s * rhoinv_s + p_s) + g3_s * (u2_s * u3_s * rhoinv_s);  // i16_flx3_s
            flx4_s = g1_s * (u3_s * u1_s * rhoinv_s) + g2_s * (u3_s * u2_s * rhoinv_s) + g3_s * (u3_s * u3_s * rhoinv_s + p_s);  // i17_flx4_s
            flx5_s = flxu_s * th_s * rhoinv_s;  // i18_flx5_s
            flx6_s = flxu_s * qt1_s * rhoinv_s;  // i19_flx6_s
            flx7_s = flxu_s * qt2_s * rhoinv_s;  // i20_flx7_s
            flx8_s = flxu_s * qt3_s * rhoinv_s;  // i21_flx8_s
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

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
    const int ii = LOCAL_ID(0);
    const int j = LOCAL_ID(1);
    const int jj = LOCAL_ID(1);
    LOCAL float D_pf[9];
    LOCAL float flx1_r_store[9];  // aliases: flx1_r_store, flx2_r_store, flx3_r_store, flx4_r_store, flx5_r_store, flx6_r_store, flx7_r_store, flx8_r_store
    LOCAL float flx1_s_store[9];  // aliases: flx1_s_store, flx2_s_store, flx3_s_store, flx4_s_store, flx5_s_store, flx6_s_store, flx7_s_store, flx8_s_store
    float tflx1_s_store;
    float tflx2_s_store;
    float tflx3_s_store;
    float tflx4_s_store;
    float tflx5_s_store;
    float tflx6_s_store;
    float tflx7_s_store;
    float tflx8_s_store;
    float flxu_r_store;
    float flxu_s_store;
    float tflxu_s_store;
    float p_r_store;
    float rhoinv_r_store;
    float rho_r_store;
    float u1_r_store;
    float u2_r_store;
    float u3_r_store;
    float th_r_store;
    float qt1_r_store;
    float qt2_r_store;
    float qt3_r_store;
    float g1_r_store;
    float g2_r_store;
    float g3_r_store;
    float g1_s_store;
    float g2_s_store;
    float g3_s_store;
    float h1_s_store;
    float h2_s_store;
    float h3_s_store;
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
        u1_r_store = q[((((e) * 2 + 0) * 3 + k) * 3 + jj) * 3 + ii].s1;  // u1_r_store_cmp
        u2_r_store = q[((((e) * 2 + 0) * 3 + k) * 3 + jj) * 3 + ii].s2;  // u2_r_store_cmp
        u3_r_store = q[((((e) * 2 + 0) * 3 + k) * 3 + jj) * 3 + ii].s3;  // u3_r_store_cmp
        g1_r_store = g[(((((e) * 3 + 0) * 3 + 0) * 3 + k) * 3 + jj) * 3 + ii];  // g1_r_store_cmp
        g2_r_store = g[(((((e) * 3 + 0) * 3 + 1) * 3 + k) * 3 + jj) * 3 + ii];  // g2_r_store_cmp
        g3_r_store = g[(((((e) * 3 + 0) * 3 + 2) * 3 + k) * 3 + jj) * 3 + ii];  // g3_r_store_cmp
        flxu_r_store = g1_r_store * u1_r_store + g2_r_store * u2_r_store + g3_r_store * u3_r_store;  // flxu_r_store_cmp
        flx1_r_store[(ii) * 3 + jj] = flxu_r_store;  // flx1_r_store_cmp
        th_r_store = q[((((e) * 2 + 1) * 3 + k) * 3 + jj) * 3 + ii].s0;  // th_r_store_cmp
        p_r_store = p0 * pow(Rgas * th_r_store / p0, gam);  // p_r_store_cmp
        rho_r_store = q[((((e) * 2 + 0) * 3 + k) * 3 + jj) * 3 + ii].s0;  // rho_r_store_cmp
        rhoinv_r_store = 1.0f / rho_r_store;  // rhoinv_r_store_cmp
        qt1_r_store = q[((((e) * 2 + 1) * 3 + k) * 3 + jj) * 3 + ii].s1;  // qt1_r_store_cmp
        qt2_r_store = q[((((e) * 2 + 1) * 3 + k) * 3 + jj) * 3 + ii].s2;  // qt2_r_store_cmp
        qt3_r_store = q[((((e) * 2 + 1) * 3 + k) * 3 + jj) * 3 + ii].s3;  // qt3_r_store_cmp
        g1_s_store = g[(((((e) * 3 + 1) * 3 + 0) * 3 + k) * 3 + jj) * 3 + ii];  // g1_s_store_cmp
        g2_s_store = g[(((((e) * 3 + 1) * 3 + 1) * 3 + k) * 3 + jj) * 3 + ii];  // g2_s_store_cmp
        g3_s_store = g[(((((e) * 3 + 1) * 3 + 2) * 3 + k) * 3 + jj) * 3 + ii];  // g3_s_store_cmp
        flxu_s_store = g1_s_store * u1_r_store + g2_s_store * u2_r_store + g3_s_store * u3_r_store;  // flxu_s_store_cmp
        flx1_s_store[(jj) * 3 + ii] = flxu_s_store;  // flx1_s_store_cmp
        h1_s_store = g[(((((e) * 3 + 2) * 3 + 0) * 3 + k) * 3 + jj) * 3 + ii];  // h1_s_store_cmp
        h2_s_store = g[(((((e) * 3 + 2) * 3 + 1) * 3 + k) * 3 + jj) * 3 + ii];  // h2_s_store_cmp
        h3_s_store = g[(((((e) * 3 + 2) * 3 + 2) * 3 + k) * 3 + jj) * 3 + ii];  // h3_s_store_cmp
        tflxu_s_store = h1_s_store * u1_r_store + h2_s_store * u2_r_store + h3_s_store * u3_r_store;  // tflxu_s_store_cmp
        tflx1_s_store = tflxu_s_store;  // tflx1_s_store_cmp
        tflx2_s_store = h1_s_store * (u1_r_store * u1_r_store * rhoinv_r_store + p_r_store) + h2_s_store * (u1_r_store * u2_r_store * rhoinv_r_store) + h3_s_store * (u1_r_store * u3_r_store * rhoinv_r_store);  // tflx2_s_store_cmp
        tflx3_s_store = h1_s_store * (u2_r_store * u1_r_store * rhoinv_r_store) + h2_s_store * (u2_r_store * u2_r_store * rhoinv_r_store + p_r_store) + h3_s_store * (u2_r_store * u3_r_store * rhoinv_r_store);  // tflx3_s_store_cmp
        tflx4_s_store = h1_s_store * (u3_r_store * u1_r_store * rhoinv_r_store) + h2_s_store * (u3_r_store * u2_r_store * rhoinv_r_store) + h3_s_store * (u3_r_store * u3_r_store * rhoinv_r_store + p_r_store);  // tflx4_s_store_cmp
        tflx5_s_store = tflxu_s_store * th_r_store * rhoinv_r_store;  // tflx5_s_store_cmp
        tflx6_s_store = tflxu_s_store * qt1_r_store * rhoinv_r_store;  // tflx6_s_store_cmp
        tflx7_s_store = tflxu_s_store * qt2_r_store * rhoinv_r_store;  // tflx7_s_store_cmp
        tflx8_s_store = tflxu_s_store * qt3_r_store * rhoinv_r_store;  // tflx8_s_store_cmp
        for (int n_f1 = 0; n_f1 < 3; ++n_f1)
        {
            BARRIER();
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f1) * 3 + i] * flx1_r_store[(n_f1) * 3 + j];  // i22_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f1) * 3 + j] * flx1_s_store[(n_f1) * 3 + i];  // i22_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = g1_r_store * (u1_r_store * u1_r_store * rhoinv_r_store + p_r_store) + g2_r_store * (u1_r_store * u2_r_store * rhoinv_r_store) + g3_r_store * (u1_r_store * u3_r_store * rhoinv_r_store);  // flx2_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = g1_s_store * (u1_r_store * u1_r_store * rhoinv_r_store + p_r_store) + g2_s_store * (u1_r_store * u2_r_store * rhoinv_r_store) + g3_s_store * (u1_r_store * u3_r_store * rhoinv_r_store);  // flx2_s_store_cmp
        for (int n_f2 = 0; n_f2 < 3; ++n_f2)
        {
            BARRIER();
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f2) * 3 + i] * flx1_r_store[(n_f2) * 3 + j];  // i23_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f2) * 3 + j] * flx1_s_store[(n_f2) * 3 + i];  // i23_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = g1_r_store * (u2_r_store * u1_r_store * rhoinv_r_store) + g2_r_store * (u2_r_store * u2_r_store * rhoinv_r_store + p_r_store) + g3_r_store * (u2_r_store * u3_r_store * rhoinv_r_store);  // flx3_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = g1_s_store * (u2_r_store * u1_r_store * rhoinv_r_store) + g2_s_store * (u2_r_store * u2_r_store * rhoinv_r_store + p_r_store) + g3_s_store * (u2_r_store * u3_r_store * rhoinv_r_store);  // flx3_s_store_cmp
        for (int n_f3 = 0; n_f3 < 3; ++n_f3)
        {
            BARRIER();
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f3) * 3 + i] * flx1_r_store[(n_f3) * 3 + j];  // i24_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f3) * 3 + j] * flx1_s_store[(n_f3) * 3 + i];  // i24_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = g1_r_store * (u3_r_store * u1_r_store * rhoinv_r_store) + g2_r_store * (u3_r_store * u2_r_store * rhoinv_r_store) + g3_r_store * (u3_r_store * u3_r_store * rhoinv_r_store + p_r_store);  // flx4_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = g1_s_store * (u3_r_store * u1_r_store * rhoinv_r_store) + g2_s_store * (u3_r_store * u2_r_store * rhoinv_r_store) + g3_s_store * (u3_r_store * u3_r_store * rhoinv_r_store + p_r_store);  // flx4_s_store_cmp
        for (int n_f4 = 0; n_f4 < 3; ++n_f4)
        {
            BARRIER();
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f4) * 3 + i] * flx1_r_store[(n_f4) * 3 + j];  // i25_rhsq_r
            rhsq[((((e) * 2 + 0) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f4) * 3 + j] * flx1_s_store[(n_f4) * 3 + i];  // i25_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = flxu_r_store * th_r_store * rhoinv_r_store;  // flx5_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = flxu_s_store * th_r_store * rhoinv_r_store;  // flx5_s_store_cmp
        for (int n_f5 = 0; n_f5 < 3; ++n_f5)
        {
            BARRIER();
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f5) * 3 + i] * flx1_r_store[(n_f5) * 3 + j];  // i26_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f5) * 3 + j] * flx1_s_store[(n_f5) * 3 + i];  // i26_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = flxu_r_store * qt1_r_store * rhoinv_r_store;  // flx6_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = flxu_s_store * qt1_r_store * rhoinv_r_store;  // flx6_s_store_cmp
        for (int n_f6 = 0; n_f6 < 3; ++n_f6)
        {
            BARRIER();
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f6) * 3 + i] * flx1_r_store[(n_f6) * 3 + j];  // i27_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f6) * 3 + j] * flx1_s_store[(n_f6) * 3 + i];  // i27_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = flxu_r_store * qt2_r_store * rhoinv_r_store;  // flx7_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = flxu_s_store * qt2_r_store * rhoinv_r_store;  // flx7_s_store_cmp
        for (int n_f7 = 0; n_f7 < 3; ++n_f7)
        {
            BARRIER();
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f7) * 3 + i] * flx1_r_store[(n_f7) * 3 + j];  // i28_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f7) * 3 + j] * flx1_s_store[(n_f7) * 3 + i];  // i28_rhsq_s
        }
        BARRIER();
        flx1_r_store[(ii) * 3 + jj] = flxu_r_store * qt3_r_store * rhoinv_r_store;  // flx8_r_store_cmp
        flx1_s_store[(jj) * 3 + ii] = flxu_s_store * qt3_r_store * rhoinv_r_store;  // flx8_s_store_cmp
        for (int n_f8 = 0; n_f8 < 3; ++n_f8)
        {
            BARRIER();
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f8) * 3 + i] * flx1_r_store[(n_f8) * 3 + j];  // i29_rhsq_r
            rhsq[((((e) * 2 + 1) * 3 + k) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + k) * 3 + j) * 3 + i] * D_pf[(n_f8) * 3 + j] * flx1_s_store[(n_f8) * 3 + i];  // i29_rhsq_s
        }
        for (int m = 0; m < 3; ++m)
        {
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx1_s_store;  // i52_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx2_s_store;  // i53_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx3_s_store;  // i54_rhsq_s
            rhsq[((((e) * 2 + 0) * 3 + m) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx4_s_store;  // i55_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s0 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx5_s_store;  // i56_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s1 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx6_s_store;  // i57_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s2 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx7_s_store;  // i58_rhsq_s
            rhsq[((((e) * 2 + 1) * 3 + m) * 3 + j) * 3 + i].s3 += Jinv[(((e) * 3 + m) * 3 + j) * 3 + i] * D_pf[(k) * 3 + m] * tflx8_s_store;  // i59_rhsq_s
        }
    }
}

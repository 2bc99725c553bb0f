//
// polyeval-b200 generated kernel: domain=i64f nvars=1 ops=8 powers=4 lanes=1
//
.version 8.7
.target sm_100a
.address_size 64

.const .align 8 .b64 pe_coef[8] = {0x4008000000000000, 0x3FF0000000000000, 0xBFF0000000000000, 0x4000000000000000, 0xC010000000000000, 0x4022000000000000, 0xC008000000000000, 0xC000000000000000};

.visible .entry pe_walk_i64f(
  .param .u64 pe_in0,
  .param .u64 pe_out0,
  .param .u64 pe_n,
  .param .u64 pe_gcoef,
  .param .u64 pe_flag,
  .param .u64 pe_bound0)
.maxntid 512, 1, 1
{
  .reg .pred %p<8>;
  .reg .b32 %r<8>;
  .reg .b64 %rd<24>;
  .reg .b64 %ix<1>;
  .reg .pred %pv<1>;
  .reg .f64 %x0_0;
  .reg .b64 %xi0_0;
  .reg .f64 %q0_0;
  .reg .f64 %q1_0;
  .reg .f64 %q2_0;
  .reg .f64 %q3_0;
  .reg .f64 %v0_0;
  .reg .f64 %v1_0;
  .reg .f64 %v2_0;
  .reg .f64 %v3_0;
  .reg .f64 %v4_0;
  .reg .f64 %v5_0;
  .reg .f64 %v6_0;
  .reg .f64 %v7_0;
  .reg .f64 %c<9>;
  .reg .b64 %tu<1>;
  mov.u32 %r1, %ctaid.x;
  mov.u32 %r2, %ntid.x;
  mov.u32 %r3, %tid.x;
  mul.wide.u32 %rd1, %r1, %r2;
  mul.lo.u64 %rd1, %rd1, 1;
  cvt.u64.u32 %rd2, %r3;
  add.u64 %rd1, %rd1, %rd2;
  ld.param.u64 %rd3, [pe_n];
  setp.ge.u64 %p1, %rd1, %rd3;
  @%p1 bra $Ldone;
  sub.u64 %rd12, %rd3, 1;
  cvt.u64.u32 %rd13, %r2;
  mul.lo.u64 %rd13, %rd13, 0;
  add.u64 %rd13, %rd1, %rd13;
  setp.lt.u64 %pv0, %rd13, %rd3;
  min.u64 %rd13, %rd13, %rd12;
  shl.b64 %ix0, %rd13, 3;
  ld.param.u64 %rd5, [pe_in0];
  cvta.to.global.u64 %rd5, %rd5;
  add.u64 %rd6, %rd5, %ix0;
  ld.global.nc.b64 %xi0_0, [%rd6];
  cvt.rn.f64.s64 %x0_0, %xi0_0;
  ld.param.u64 %rd8, [pe_bound0];
  abs.s64 %rd9, %xi0_0;
  setp.gt.u64 %p2, %rd9, %rd8;
  @!%p2 bra $Lbok0;
  ld.param.u64 %rd7, [pe_flag];
  cvta.to.global.u64 %rd7, %rd7;
  @%pv0 st.global.u32 [%rd7], 1;
$Lbok0:
  mov.f64 %q0_0, %x0_0;
  mul.rn.f64 %q1_0, %q0_0, %q0_0;
  mul.rn.f64 %q2_0, %q1_0, %q1_0;
  mul.rn.f64 %q3_0, %q2_0, %q2_0;
  ld.const.f64 %c0, [pe_coef+0];
  ld.const.f64 %c1, [pe_coef+8];
  fma.rn.f64 %v0_0, %c0, %q3_0, %c1;
  ld.const.f64 %c2, [pe_coef+16];
  ld.const.f64 %c3, [pe_coef+24];
  fma.rn.f64 %v1_0, %c2, %q0_0, %c3;
  ld.const.f64 %c4, [pe_coef+32];
  fma.rn.f64 %v2_0, %v1_0, %q1_0, %c4;
  ld.const.f64 %c5, [pe_coef+8];
  fma.rn.f64 %v3_0, %c5, %q0_0, %v2_0;
  fma.rn.f64 %v4_0, %v3_0, %q2_0, %v0_0;
  ld.const.f64 %c6, [pe_coef+40];
  ld.const.f64 %c7, [pe_coef+48];
  fma.rn.f64 %v5_0, %c6, %q0_0, %c7;
  fma.rn.f64 %v6_0, %v5_0, %q1_0, %v4_0;
  ld.const.f64 %c8, [pe_coef+56];
  fma.rn.f64 %v7_0, %c8, %q0_0, %v6_0;
  ld.param.u64 %rd9, [pe_out0];
  cvta.to.global.u64 %rd9, %rd9;
  cvt.rni.s64.f64 %tu0, %v7_0;
  add.u64 %rd10, %rd9, %ix0;
  @%pv0 st.global.b64 [%rd10], %tu0;
$Ldone:
  ret;
}

